#!/bin/bash
# round-2: per-polynomial affine fetch offsets (sorted mode) vs offset tables; class-major table loop on c3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python tools/variants.py c3 --only default,offt_table,cm3_tl_b512_t2048,cm3_tl_b256_t2048,cm3_tl_b512_t1536,cm3_tl_b384_t1536,cm3_tl_b640_t1920,cm3_tl_b512_t2048_c42,tl_b512_t2048 --reps 20 2>&1 | tee gpurun_out/r02d_variants_c3.txt
timeout 900 python tools/variants.py c4v --only default,offt_table --reps 10 2>&1 | tee gpurun_out/r02d_variants_c4v.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "voronoi3 and (sorted or radix or presort)" > gpurun_out/r02d_pytest.log 2>&1; tail -3 gpurun_out/r02d_pytest.log
