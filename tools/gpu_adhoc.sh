mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_render.py -x -q 2>&1 | tail -3
for c in c3r c3rs; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 10 2>&1 | grep -E "Gsamples|FAIL|Error"; done
