#!/bin/bash
# quick GPU session: build+smoke, gpu tests, variant timings, launch list of the binned path
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 600 python tools/variants.py ${1:-c2} 2>&1 | grep -E "Grecon|FAIL|Error" 
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_variants.csv python tools/variants.py ${1:-c2} --only binned_tma_b256_loop --reps 2 > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open("gpurun_out/launches_variants.csv")))
hdr=rows[0]
ki=hdr.index("Kernel Name"); vi=hdr.index("Metric Value")
for r in rows[1:][-12:]:
    print(f"{r[ki][:40]:40s} {r[vi]}")
PY
