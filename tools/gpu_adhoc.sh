mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "radix" 2>&1 | tail -2
for c in c3 c5 c4v; do echo "== $c"; for v in default radix; do timeout 600 python tools/variants.py $c --reps 10 --only $v 2>&1 | grep -E "Grecon|FAIL|Error"; done; done
