#!/bin/bash
# sorted-kernel shared tables read from global memory (gtables knob): c3 and c5
mkdir -p gpurun_out
EX="$(cat tools/sweep_c3_shapes.json)"
timeout 600 python tools/variants.py c3 --reps 20 --extra "$EX" --only default,gT,gTA,gTAP,gTA_b576_t3456 > gpurun_out/r02g_variants_c3_gtables.txt 2>&1
timeout 900 python tools/variants.py c5 --reps 5 --extra "$EX" --only default,gT,gTA,gTAP > gpurun_out/r02g_variants_c5_gtables.txt 2>&1
cat gpurun_out/r02g_variants_c3_gtables.txt gpurun_out/r02g_variants_c5_gtables.txt
for v in gTAP; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sg_eval_kernel -s 2 -c 1 \
    -o gpurun_out/prof_c3_$v -f python tools/variants.py c3 --extra "$EX" --only $v --reps 2 > /dev/null 2>&1
done
