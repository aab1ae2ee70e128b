#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tools/variants.py c4v --only default,v_b640_t1280,v_b640_t1280_cm3,v_b640_t1280_p32,v_b640_t1280_p16,v_b704_t1408,v_b576_t1152,v_b640_t1280_horner --reps 10 2>&1 | tee gpurun_out/r02t_c4v.txt
