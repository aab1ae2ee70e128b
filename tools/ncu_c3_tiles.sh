#!/bin/bash
# ncu --set full of the c3 sorted kernel at three tile shapes (the 3,840-query cliff)
mkdir -p gpurun_out
EX="$(cat tools/sweep_c3_shapes.json)"
for v in default t3840 b608_t3648; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sg_eval_kernel -s 2 -c 1 \
    -o gpurun_out/prof_c3_$v -f python tools/variants.py c3 --extra "$EX" --only $v --reps 2 > /dev/null 2>&1
  ls -la gpurun_out/prof_c3_$v.ncu-rep
done
