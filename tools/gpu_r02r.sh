#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/variants.py c4 --only default,c4_table,c4_table_b256,c4_lut,c4_tloop,c4_sites,c4_b64,c4_b128_mb8 --reps 20 2>&1 | tee gpurun_out/r02r_c4.txt
