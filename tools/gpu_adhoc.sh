mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in c2 c1 c3 c4 c4v; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 20 --only default 2>&1 | grep -E "Grecon|FAIL|Error"; done
