mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "pack2" 2>&1 | tail -3
for c in c2 c1 c4 c4v; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 20 --only pack2 2>&1 | grep -E "Grecon|FAIL|Error"; timeout 600 python tools/variants.py $c --reps 20 --only default 2>&1 | grep -E "Grecon|FAIL|Error"; done
