mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/tests.txt; cat gpurun_out/tests.txt
for c in c4 c4v c3; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 20 --only default 2>&1 | grep -E "Grecon|FAIL|Error"; done
