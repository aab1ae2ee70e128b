mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_render.py tests/test_capi.py -x -q 2>&1 | tail -4
for c in c3r c3rs; do timeout 600 python bench.py --config $c --steps 20 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 1500 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err; done
