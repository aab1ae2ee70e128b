#!/bin/bash
# Round-2 evidence pass (run under gpurun from the repo root):
# build + smoke, the GPU test suite, then tools/gpu_round.sh for the given configs.
# usage: bash tools/gpu_r02.sh <tag> "<configs>" [tests=1]
TAG=${1:-r02}; CFGS=${2:-c5 c3 c4v c4v4 c2 c4 c1 c5u c3r c3rs}; TESTS=${3:-1}
mkdir -p gpurun_out
nvidia-smi -L
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -2 gpurun_out/${TAG}_smoke.log
if [ "$TESTS" = "1" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1; tail -5 gpurun_out/${TAG}_pytest_gpu.log
fi
bash tools/gpu_round.sh $TAG "$CFGS"
