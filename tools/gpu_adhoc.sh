mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
echo "== variants c4v"; timeout 600 python tools/variants.py c4v --reps 10 2>&1 | grep -E "Grecon|FAIL|Error"
