#!/bin/bash
# round-2: chunk-local presort (sort key = (chunk of the original index, bin))
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "presort" > gpurun_out/r02e_pytest.log 2>&1; tail -3 gpurun_out/r02e_pytest.log
timeout 900 python tools/variants.py c4v --only default,ch18,ch19,ch20,ch21,ch22,pre8_ch20,pre32_ch20 --reps 10 2>&1 | tee gpurun_out/r02e_variants_c4v.txt
timeout 900 python tools/variants.py c4 --only default,c4_srt_pre16_ch20,c4_srt_pre16_ch21,c4_srt_sym_pre16_ch20,c4_srt_pre8_ch20 --reps 10 2>&1 | tee gpurun_out/r02e_variants_c4.txt
timeout 900 python tools/variants.py c5u --only default,ch22,ch24 --reps 3 2>&1 | tee gpurun_out/r02e_variants_c5u.txt
