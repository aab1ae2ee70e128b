mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q -k "binned or c1 or c2 or kat" 2>&1 | tail -2
for c in c2 c1; do echo "== $c"; timeout 600 python tools/variants.py $c --reps 30 --only default 2>&1 | grep -E "Grecon|FAIL|Error"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_r01e.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
