#!/bin/bash
# One gpurun session: build, smoke, GPU tests, bench, ncu launch list + one full capture.
# usage (from the repo root, under gpurun): bash tools/gpu_check.sh <config> <tag> [tests]
set -x
CFG=${1:-c2}; TAG=${2:-r01}; TESTS=${3:-1}
mkdir -p gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
if [ "$TESTS" = "1" ]; then timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15; fi
timeout 600 python bench.py --config $CFG --steps 300 --no-cpu > gpurun_out/bench_${CFG}_${TAG}.json 2> gpurun_out/bench_${CFG}_${TAG}.err; tail -c 3000 gpurun_out/bench_${CFG}_${TAG}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${TAG}.csv python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sg_eval -s 3 -c 1 -o gpurun_out/prof_${CFG}_${TAG} -f python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_${CFG}_${TAG}.log 2>&1
ls -la gpurun_out
