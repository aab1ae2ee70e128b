#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tools/variants.py c4v --only default,v_b512_t1024,v_b512_t1024_cm3,v_b256_t1024,v_b256_t512,v_b384_t1152,v_b640_t1280,v_b512_t512_cm3 --reps 10 2>&1 | tee gpurun_out/r02s_c4v.txt
