#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/variants.py c3 --only default,cm4,cm4_t2560,cm4_t3840,cm4_b512_t3072 --reps 20 2>&1 | tee gpurun_out/r02m_variants_c3.txt
