#!/bin/bash
mkdir -p gpurun_out
python tools/micro/pcie_bw.py > gpurun_out/r02_pcie_bw.json 2>&1; cat gpurun_out/r02_pcie_bw.json
bash tools/gpu_round.sh r02c "c4v c4v4"
