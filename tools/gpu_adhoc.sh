mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q -k "binned or c1 or c2 or kat or c5" 2>&1 | tail -2
for c in c2 c1; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 30 --only default 2>&1 | grep -E "Grecon|FAIL|Error"; done
for c in c4v c4; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 10 --only l1_bin104 2>&1 | grep -E "Grecon|FAIL|Error"; done
echo "== c5u"; timeout 600 python tools/variants.py c5u --reps 3 --only default 2>&1 | grep -E "Grecon|FAIL|Error"
