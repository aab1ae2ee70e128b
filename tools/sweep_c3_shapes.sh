mkdir -p gpurun_out
EX="$(cat tools/sweep_c3_shapes.json)"
timeout 900 python tools/variants.py c3 --reps 20 --extra "$EX" --only default,b576_t2880,b576_t3456,b608_t3040,b672_t3360,b544_t3264,b320_t1600_mb2,b320_t1920_mb2,b352_t1760_mb2,b288_t1728_mb2,b608_t3648,b544_t3808,b640_t3200_cs > gpurun_out/r02g_variants_c3_shapes.txt 2>&1
cat gpurun_out/r02g_variants_c3_shapes.txt
