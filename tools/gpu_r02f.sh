#!/bin/bash
# round-2: two pairs per thread in packed FFMA2 (sorted mode, immediates, class-major chunks)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "pairs or (values_f32 and (34 or 35 or 36))" > gpurun_out/r02f_pytest.log 2>&1; tail -5 gpurun_out/r02f_pytest.log
timeout 1200 python tools/variants.py c3 --only default,pp_b384_t2304,pp_b384_t1536,pp_b256_t2048,pp_b320_t2560,pp_b512_t2048 --reps 20 2>&1 | tee gpurun_out/r02f_variants_c3.txt
timeout 900 python tools/variants.py c4v --only default,pp_cm3_b256,pp_cm3_b384,pp_cm3_b256_horner --reps 10 2>&1 | tee gpurun_out/r02f_variants_c4v.txt
