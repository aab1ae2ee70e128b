#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python tools/variants.py c4v4 --only default,v4_p64,v4_p16,v4_b384,v4_b512,v4_b256_t512,v4_cm3 --reps 5 2>&1 | tee gpurun_out/r02u_c4v4.txt
