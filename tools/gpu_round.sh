#!/bin/bash
# Per bench configuration, on one B200 (run under gpurun from the repo root):
#   1. the launch list of one bench step (ncu, per-kernel time + DRAM bytes),
#   2. one `ncu --set full` capture of the evaluation kernel, summarised on the box into
#      profiles/ncu_<config>.json (read by bench.py's roofline block) and a text summary,
#   3. the bench line itself (after the profile, so its executed/issue figures are current).
# usage: bash tools/gpu_round.sh <tag> "<configs>"
TAG=${1:-r02}; CFGS=${2:-c5 c3 c2 c1 c4 c4v c4v4 c3r c3rs c5u}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for c in $CFGS; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/${TAG}_launches_${c}.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:sg_eval_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${c}_${TAG} -f python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_${c}_${TAG}.log 2>&1
  python tools/ncu_extract.py $c gpurun_out/prof_${c}_${TAG}.ncu-rep $TAG > /dev/null 2>&1 && cp profiles/ncu_${c}.json gpurun_out/
  python tools/ncu_summary.py gpurun_out/prof_${c}_${TAG}.ncu-rep > gpurun_out/${TAG}_ncu_${c}_summary.txt 2>&1
  rm -f gpurun_out/prof_${c}_${TAG}.ncu-rep   # gpurun copies back <= 64 MiB: keep the summaries only
  timeout 1200 python bench.py --config $c > gpurun_out/${TAG}_bench_${c}.json 2> gpurun_out/${TAG}_bench_${c}.err
  echo "$c: $(head -c 300 gpurun_out/${TAG}_bench_${c}.json)"
done
