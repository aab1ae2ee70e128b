#!/bin/bash
# quick GPU session: build+smoke, gpu tests, variant timings, launch list of the binned path
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 600 python tools/variants.py ${1:-c2} 2>&1 | grep -E "Grecon|FAIL|Error" 
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_variants.csv python tools/variants.py ${1:-c2} --only default --reps 2 > /dev/null 2>&1
python - <<'PY'
import csv
lines=open("gpurun_out/launches_variants.csv").read().splitlines()
i=[k for k,l in enumerate(lines) if l.startswith('"ID"')][0]
rows=list(csv.reader(lines[i:]))
hdr=rows[0]
ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value")
for r in rows[1:][-12:]:
    print(f"{r[ki][:40]:40s} {r[vi]}")
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sg_eval_kernel -s 2 -c 1 -o gpurun_out/prof_binned -f python tools/variants.py ${1:-c2} --only default --reps 2 > /dev/null 2>&1
ls -la gpurun_out/prof_binned.ncu-rep
