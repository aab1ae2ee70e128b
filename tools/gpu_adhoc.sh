mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q -k "binned or c1 or c2 or kat" 2>&1 | tail -2
for cfg in c2 c1; do
  echo "== $cfg default"; timeout 300 python tools/variants.py $cfg --reps 30 --only default 2>&1 | grep -E "Grecon|FAIL|Error"
  echo "== $cfg 512x2"; SPLINEGPU_SCATTER_THREADS=512 SPLINEGPU_SCATTER_GROUPS=2 timeout 300 python tools/variants.py $cfg --reps 30 --only default 2>&1 | grep -E "Grecon|FAIL|Error"
  echo "== $cfg 256x4"; SPLINEGPU_SCATTER_THREADS=256 SPLINEGPU_SCATTER_GROUPS=4 timeout 300 python tools/variants.py $cfg --reps 30 --only default 2>&1 | grep -E "Grecon|FAIL|Error"
done
SPLINEGPU_SCATTER_THREADS=512 SPLINEGPU_SCATTER_GROUPS=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "binned" 2>&1 | tail -1
