mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for cfg in c1; do
for th in 1024 512 256; do for mp in 4096 8192 16384 32768; do
  echo "== $cfg scatter threads $th minper $mp"
  SPLINEGPU_SCATTER_THREADS=$th SPLINEGPU_SORT_MINPER=$mp SPLINEGPU_SORT_CTAS=4 timeout 300 python tools/variants.py $cfg --reps 50 --only default 2>&1 | grep -E "Grecon|FAIL|Error"
done; done; done
