#!/bin/bash
# official-style bench lines for the configs + launch list + one full ncu capture of the default
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
TAG=${1:-r01}
for c in ${2:-c2 c1 c3 c4}; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_${TAG}.json 2> gpurun_out/bench_${c}_${TAG}.err
  tail -c 2500 gpurun_out/bench_${c}_${TAG}.json; echo; tail -3 gpurun_out/bench_${c}_${TAG}.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2_${TAG}.csv python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sg_eval_kernel -s 3 -c 1 -o gpurun_out/prof_c2_${TAG} -f python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out | tail -12
