#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/variants.py c3 --only default,t3840,t4480,b512_t4096,b576_t4032,b704_t3520 --reps 20 2>&1 | tee gpurun_out/r02j_variants_c3.txt
