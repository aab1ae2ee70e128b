#!/bin/bash
bash tools/gpu_round.sh r02d "c4v c4v4"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "qhoist or 39 or 40 or c4v" > gpurun_out/r02d_pytest.log 2>&1; tail -3 gpurun_out/r02d_pytest.log
