#!/bin/bash
# round-2: binned TMA bricks for c4 (4 cosets, 8-cell bins -> 9261 bins), tiled scatter beyond 2048 bins
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
V="default,c4_bin8_b256,c4_bin8_b128,c4_bin8_b512_sym,c4_bin8_b256_sym,c4_bin8_b256_branchy"
timeout 900 python tools/variants.py c4 --only $V --reps 10 2>&1 | tee gpurun_out/r02i_variants_c4.txt
SPLINEGPU_TILED_MAX_BINS=10240 timeout 900 python tools/variants.py c4 --only $V --reps 10 2>&1 | tee gpurun_out/r02i_variants_c4_tiled.txt
SPLINEGPU_TILED_MAX_BINS=10240 timeout 900 python tools/variants.py c4v --only default,pre8 --reps 10 2>&1 | tee gpurun_out/r02i_variants_c4v_tiled.txt
timeout 900 python tools/variants.py c3 --only default,c3_sym,c3_sites --reps 10 2>&1 | tee gpurun_out/r02i_variants_c3.txt
