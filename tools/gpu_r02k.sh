#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/variants.py c3 --only default,t2560,t1920,radix0,radix0_smem,radix0_smem_t2560 --reps 20 2>&1 | tee gpurun_out/r02k_variants_c3.txt
