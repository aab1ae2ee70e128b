mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_kat.py tests/test_render.py -x -q -k "sorted" 2>&1 | tail -2
for c in c3 c5; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 10 --only default 2>&1 | grep -E "Grecon|FAIL|Error"; timeout 600 python tools/variants.py $c --reps 10 --only nopf 2>&1 | grep -E "Grecon|FAIL|Error"; timeout 600 python tools/variants.py $c --reps 10 --only pf_ 2>&1 | grep -E "Grecon|FAIL|Error"; done
echo "== c3r"; timeout 600 python tools/variants.py c3r --reps 10 --only sorted_b512_t1536 2>&1 | grep -E "Gsamples|FAIL|Error"
