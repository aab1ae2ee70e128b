#!/bin/bash
# ncu evidence for every bench configuration (run under gpurun from the repo root):
# launch list of one bench step (per-kernel times + DRAM bytes) and one --set full capture
# of the evaluation kernel, both from `bench.py --config <c>` itself.
# usage: bash tools/gpu_profiles.sh <tag> [configs]
TAG=${1:-r01}; CFGS=${2:-c2 c1 c3 c4 c4v}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for c in $CFGS; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${c}_${TAG}.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sg_eval_kernel -s 3 -c 1 \
    -o gpurun_out/prof_${c}_${TAG} -f python bench.py --config $c --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_${c}_${TAG}.log 2>&1
done
ls -la gpurun_out | tail -20
