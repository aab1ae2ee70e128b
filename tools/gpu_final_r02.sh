#!/bin/bash
# round-2 final pass: build + smoke, the full -m gpu suite, the default bench line, the reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1; tail -3 gpurun_out/r02_final_smoke.log
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_final_pytest_gpu.log 2>&1; tail -4 gpurun_out/r02_final_pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/r02_final_bench.json 2> gpurun_out/r02_final_bench.err; tail -c 300 gpurun_out/r02_final_bench.json
timeout 900 python bench.py --impl reference > gpurun_out/r02_final_bench_reference.json 2> gpurun_out/r02_final_bench_reference.err; tail -c 300 gpurun_out/r02_final_bench_reference.json
