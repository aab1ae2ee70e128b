#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in default t2560; do
  timeout 900 ncu --set full --clock-control none -k regex:sg_eval_kernel -s 2 -c 1 -o gpurun_out/tile_$v -f python tools/variants.py c3 --only $v --reps 2 > /dev/null 2>&1
done
python tools/ncu_summary.py --table gpurun_out/tile_default.ncu-rep gpurun_out/tile_t2560.ncu-rep > gpurun_out/r02l_tile.txt 2>&1
ncu -i gpurun_out/tile_default.ncu-rep --page raw --csv > gpurun_out/r02l_raw_default.csv 2>/dev/null
ncu -i gpurun_out/tile_t2560.ncu-rep --page raw --csv > gpurun_out/r02l_raw_t2560.csv 2>/dev/null
rm -f gpurun_out/tile_*.ncu-rep
cat gpurun_out/r02l_tile.txt
