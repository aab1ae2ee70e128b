#!/bin/bash
# sorted kernel: psi order alternating per tile (cflip) on c3 / c5, and its GPU parity cases
mkdir -p gpurun_out
EX="$(cat tools/sweep_c3_shapes.json)"
timeout 600 python tools/variants.py c3 --reps 20 --extra "$EX" --only default,cflip,cflip_gT,default_again,cflip_again > gpurun_out/r02g_variants_c3_cflip.txt 2>&1
timeout 900 python tools/variants.py c5 --reps 5 --extra "$EX" --only default,cflip,cflip_gT,default_again,cflip_again > gpurun_out/r02g_variants_c5_cflip.txt 2>&1
cat gpurun_out/r02g_variants_c3_cflip.txt gpurun_out/r02g_variants_c5_cflip.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "f32_vs_reference and 37-" -p no:cacheprovider > gpurun_out/r02g_cflip_parity.log 2>&1; tail -2 gpurun_out/r02g_cflip_parity.log
