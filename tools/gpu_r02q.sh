#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/variants.py c3r --only march,r_cm3_b640_t3200,r_cm3_b512_t3072,r_cm3_b512_t2048,r_cm3_b384_t2304 --reps 20 2>&1 | tee gpurun_out/r02q_c3r.txt
