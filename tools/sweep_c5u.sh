#!/bin/bash
# c5u: locality pre-sort bin edge with the tiled scatter allowed up to 10,240 bins
mkdir -p gpurun_out
EX="$(cat tools/sweep_c5u.json)"
export SPLINEGPU_TILED_MAX_BINS=10240
timeout 1200 python tools/variants.py c5u --reps 3 --extra "$EX" --only default,pre20,pre24,pre32,pre40,pre48 > gpurun_out/r02g_variants_c5u_presort.txt 2>&1
cat gpurun_out/r02g_variants_c5u_presort.txt
