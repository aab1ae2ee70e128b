#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c4v c4v4 c3 c5u; do timeout 600 python tools/diag_pou.py $c; done 2>&1 | tee gpurun_out/r02_diag_pou.txt
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu_full.log 2>&1
tail -40 gpurun_out/r02_pytest_gpu_full.log
