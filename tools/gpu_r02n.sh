#!/bin/bash
# sort scatter launch-shape sweep (env knobs of the C ABI) on c2 and c4v
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in c2 c4v c5u; do
for env in "X=0" "SPLINEGPU_SCATTER_GROUPS=2" "SPLINEGPU_SCATTER_THREADS=256 SPLINEGPU_SCATTER_GROUPS=4" "SPLINEGPU_SCATTER_THREADS=1024" "SPLINEGPU_SORT_CTAS=1" "SPLINEGPU_SORT_CTAS=4" "SPLINEGPU_SORT_CTAS=4 SPLINEGPU_SCATTER_GROUPS=2"; do
  st=100; [ $cfg = c5u ] && st=5
  r=$(env $env timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['kernel']['eval_kernel_ms'])")
  echo "$cfg $env: $r" | tee -a gpurun_out/r02n_sort_env.txt
done; done
