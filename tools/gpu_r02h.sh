#!/bin/bash
# round-2: full GPU suite, knob counter pairs, c4v presort choice, ncu of the sort scatter
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; tail -2 gpurun_out/r02h_smoke.log
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02h_pytest_gpu.log 2>&1; tail -8 gpurun_out/r02h_pytest_gpu.log
timeout 900 python tools/variants.py c4v --only default,srt_sym_pre32,srt_sym_pre64,cm3_sym_pre32,pre8 --reps 10 2>&1 | tee gpurun_out/r02h_variants_c4v.txt
for c in c2 c4v; do
  timeout 900 ncu --set full --clock-control none -k regex:sg_bin_scatter -s 1 -c 1 -o gpurun_out/scat_$c -f python bench.py --config $c --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/scat_$c.ncu-rep > gpurun_out/r02h_ncu_scatter_$c.txt 2>&1; rm -f gpurun_out/scat_$c.ncu-rep
  head -30 gpurun_out/r02h_ncu_scatter_$c.txt
done
bash tools/gpu_knobs.sh r02
