#!/bin/bash
# Full status pass on one B200: build, smoke, GPU tests, bench lines for every config
# (+ the reference arm once).  usage (under gpurun, from the repo root):
#   bash tools/gpu_status.sh <tag> [configs] [variants: 0|1]
TAG=${1:-r01}; CFGS=${2:-c2 c1 c3 c4 c4v}; VAR=${3:-0}
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in $CFGS; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err
  tail -c 300 gpurun_out/bench_${c}_${TAG}.json; echo; tail -2 gpurun_out/bench_${c}_${TAG}.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
tail -c 400 gpurun_out/bench_ref_${TAG}.json
if [ "$VAR" = "1" ]; then
  for c in $CFGS; do echo "== variants $c"; timeout 600 python tools/variants.py $c --reps 20 2>&1 | grep -E "Grecon|FAIL|Error"; done
fi
