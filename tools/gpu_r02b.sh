#!/bin/bash
# round-2: FCC order-3 Voronoi space fix on the GPU (parity + full-size), c4v bench, c4 locality variants
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fcc_voronoi3 or c4v or linfetch or partition" > gpurun_out/r02b_pytest.log 2>&1
tail -5 gpurun_out/r02b_pytest.log
timeout 900 python tools/variants.py c4 --only default,c4_l1_bin16,c4_l1_bin32,c4_l1_bin32_b128,c4_srt_pre16,c4_srt_pre32,c4_srt_sym_pre16,c4_srt_sym_pre32,c4_sym --reps 20 2>&1 | tee gpurun_out/r02b_variants_c4.txt
timeout 900 python tools/variants.py c4v --only default,srt_sym_pre16,srt_sym_pre32,srt_sym_pre64,srt_pre16,tlc_b256_pre32,cm3_sym_pre32,srt_sym --reps 10 2>&1 | tee gpurun_out/r02b_variants_c4v.txt
timeout 900 python bench.py --config c4v --steps 100 > gpurun_out/r02b_bench_c4v.json 2> gpurun_out/r02b_bench_c4v.err; tail -c 600 gpurun_out/r02b_bench_c4v.json
