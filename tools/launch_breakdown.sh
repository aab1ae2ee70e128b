python -c "import __graft_entry__ as g; g.build()"
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2_sym.csv python tools/variants.py c2 --only default --reps 2 > /dev/null 2>&1
python - <<'PY'
import csv, collections
lines=open("gpurun_out/launches_c2_sym.csv").read().splitlines()
i=[k for k,l in enumerate(lines) if l.startswith('"ID"')][0]
rows=list(csv.reader(lines[i:])); hdr=rows[0]
ki=hdr.index("Kernel Name"); mi=hdr.index("Metric Name"); vi=hdr.index("Metric Value"); ii=hdr.index("ID")
per=collections.defaultdict(dict); names={}
for r in rows[1:]:
    per[int(r[ii])][r[mi]]=r[vi]; names[int(r[ii])]=r[ki]
for k in sorted(per)[-10:]:
    print(names[k][:30], per[k].get('gpu__time_duration.sum'), per[k].get('dram__bytes_read.sum'), per[k].get('dram__bytes_write.sum'))
PY
timeout 900 python bench.py --config c2 > gpurun_out/bench_c2_sym.json 2>&1; tail -c 3000 gpurun_out/bench_c2_sym.json
