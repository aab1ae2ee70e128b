mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for cv in "c3 default" "c3 sorted_b512" "c4 sorted_b512" "c2 default"; do
  set -- $cv
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sg_eval_kernel -s 1 -c 1 -o gpurun_out/prof_$1_$2_int -f python tools/variants.py $1 --only $2 --reps 1 > /dev/null 2>&1
done
ls -la gpurun_out/*.ncu-rep
