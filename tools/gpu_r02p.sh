#!/bin/bash
# refresh the c4v evidence (presort 64) + the default bench line end to end
mkdir -p gpurun_out
bash tools/gpu_round.sh r02c "c4v"
timeout 1500 python bench.py > gpurun_out/r02c_bench_default.json 2> gpurun_out/r02c_bench_default.err
tail -c 400 gpurun_out/r02c_bench_default.json
