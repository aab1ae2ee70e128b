mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for c in c4 c4v c3 c2 c1; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 20 --only stream 2>&1 | grep -E "Grecon|FAIL|Error"; timeout 600 python tools/variants.py $c --reps 20 --only default 2>&1 | grep -E "Grecon|FAIL|Error"; done
