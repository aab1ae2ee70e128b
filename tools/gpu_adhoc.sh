mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for c in c4 c4v; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 10 --only occ 2>&1 | grep -E "Grecon|FAIL|Error"; done
for c in c4v; do echo "== $c table"; for v in occ_128x8 occ_256x4; do :; done; done
echo "== c3"; timeout 600 python tools/variants.py c3 --reps 10 --only sorted_b 2>&1 | grep -E "Grecon|FAIL|Error"
