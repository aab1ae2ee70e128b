#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/variants.py c5u --only default,u_cm3_pre32,u_cm3_pre136 --reps 3 2>&1 | tee gpurun_out/r02o_c5u.txt
SPLINEGPU_TILED_MAX_BINS=4096 timeout 900 python tools/variants.py c5u --only default,u_cm3_pre32 --reps 3 2>&1 | tee -a gpurun_out/r02o_c5u.txt
