#!/bin/bash
# ncu --set full of one variant's evaluation kernel: bash tools/ncu_one.sh <config> <variant> <tag>
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sg_eval_kernel -s 2 -c 1 -o gpurun_out/prof_$3 -f python tools/variants.py $1 --only $2 --reps 2 > /dev/null 2>&1
ls -la gpurun_out/prof_$3.ncu-rep
