#!/bin/bash
# round-2: c4v presort choice; c3 sorted-kernel SASS region profile (where the non-FP issue goes)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/variants.py c4v --only default,nopre,nopre_b256,nopre_horner,nopre_cm3,nopre_cm3_b640_t3200,pre8 --reps 10 2>&1 | tee gpurun_out/r02c_variants_c4v.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sg_eval_kernel -s 2 -c 1 -o gpurun_out/prof_c3_r02c -f python tools/variants.py c3 --only default --reps 2 > /dev/null 2>&1
python tools/sass_profile.py gpurun_out/prof_c3_r02c.ncu-rep 40 > gpurun_out/r02c_c3_regions.txt 2>&1
head -60 gpurun_out/r02c_c3_regions.txt
ncu -i gpurun_out/prof_c3_r02c.ncu-rep --page source --csv --print-source sass > gpurun_out/r02c_c3_sass.csv 2>/dev/null
gzip -f gpurun_out/r02c_c3_sass.csv; rm -f gpurun_out/prof_c3_r02c.ncu-rep
ls -la gpurun_out
