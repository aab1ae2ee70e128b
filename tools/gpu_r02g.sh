#!/bin/bash
# round-2 evidence pass: smoke, full GPU suite, then per config launch list + ncu capture + bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02g_smoke.log 2>&1; tail -2 gpurun_out/r02g_smoke.log
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02g_pytest_gpu.log 2>&1; tail -8 gpurun_out/r02g_pytest_gpu.log
bash tools/gpu_round.sh r02b "c5 c3 c2 c1 c4 c4v c4v4 c5u c3r c3rs"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b_bench_reference.json 2> gpurun_out/r02b_bench_reference.err
tail -c 300 gpurun_out/r02b_bench_reference.json
