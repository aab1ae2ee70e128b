mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_kat.py -x -q -k "sorted or presort or radix or unreachable" 2>&1 | tail -2
echo "== c5u"; for v in default presort136 presort68; do timeout 900 python tools/variants.py c5u --reps 3 --only $v 2>&1 | grep -E "Grecon|FAIL|Error"; done
echo "== c3"; timeout 900 python tools/variants.py c3 --reps 10 --only default 2>&1 | grep -E "Grecon|FAIL|Error"
echo "== c5"; timeout 900 python tools/variants.py c5 --reps 3 --only default 2>&1 | grep -E "Grecon|FAIL|Error"
