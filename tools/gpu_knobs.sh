#!/bin/bash
# ncu --set full counter pairs for the paper's knobs (north_star: "ncu counters evidence each
# choice"): one capture per (config, variant), summarised side by side per knob.
# usage (under gpurun, repo root): bash tools/gpu_knobs.sh <tag>
TAG=${1:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cap() {  # config variant
  timeout 900 ncu --set full --clock-control none -k regex:sg_eval_kernel -s 2 -c 1 \
    -o gpurun_out/knob_${TAG}_$1_$2 -f python tools/variants.py $1 --only $2 --reps 2 > gpurun_out/knob_${TAG}_$1_$2.log 2>&1
}
# dispatch: predicated vs branchy (FCC 6-dir box, K = 3, direct mode)
cap c4 c4_direct_b128; cap c4 c4_branchy
# polynomial form: greedy Horner vs symmetry-reduced (BCC quintic box, binned/TMA)
cap c2 horner; cap c2 default
# coefficient storage: FMA immediates vs shared-memory table (BCC quintic box, binned/TMA)
cap c2 table
# fetch: TMA-staged bricks vs L1/L2 gathers (binned sort kept) vs unsorted direct gathers
cap c2 binned_l1; cap c2 direct
# Voronoi dispatch: predicated direct vs psi-sorted (order-2 BCC Voronoi, rays)
cap c3o2 direct; cap c3o2 srt_imm
# sorted-mode fetch offsets: per-polynomial affine vs per-site offset table (order-3 BCC Voronoi)
cap c3 default; cap c3 offt_table
for k in "dispatch:c4_c4_direct_b128 c4_c4_branchy" "form:c2_horner c2_default" \
         "coeffs:c2_default c2_table" "fetch:c2_default c2_binned_l1 c2_direct" \
         "voronoi_dispatch:c3o2_direct c3o2_srt_imm" "fetch_offsets:c3_default c3_offt_table"; do
  name=${k%%:*}; reps=""
  for v in ${k#*:}; do reps="$reps gpurun_out/knob_${TAG}_$v.ncu-rep"; done
  python tools/ncu_summary.py --table $reps > gpurun_out/${TAG}_knob_${name}.txt 2>&1
done
rm -f gpurun_out/knob_${TAG}_*.ncu-rep   # gpurun copies back <= 64 MiB
ls gpurun_out | grep knob
