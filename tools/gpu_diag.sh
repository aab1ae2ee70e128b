#!/bin/bash
# round-2 diagnostics: tcgen05 micro-test, partition-of-unity over variants, full GPU suite
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
(cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_tf32 tc_tf32.cu && timeout 120 ./tc_tf32) > gpurun_out/r02_tc_tf32.txt 2>&1
cat gpurun_out/r02_tc_tf32.txt
for c in ${1:-c4v c4v4 c3 c5u}; do timeout 600 python tools/diag_pou.py $c; done 2>&1 | tee gpurun_out/r02_diag_pou.txt
if [ "${2:-1}" = "1" ]; then
  timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu_full.log 2>&1
  tail -30 gpurun_out/r02_pytest_gpu_full.log
fi
