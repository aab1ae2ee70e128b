#!/bin/bash
# compute-sanitizer memcheck + racecheck (+ synccheck) over one launch per execution mode;
# logs in gpurun_out/sanitize_<tool>_<mode>.log.  usage: bash tools/gpu_sanitize.sh ["modes"]
mkdir -p gpurun_out
for mode in ${1:-direct binned sorted sorted_table presort_grad render}; do
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $mode \
      > gpurun_out/sanitize_${tool}_${mode}.log 2>&1
    echo "$tool $mode rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${mode}.log | tail -1)"
  done
done
