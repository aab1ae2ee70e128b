"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum[,dram...]):
the timed bench step's kernels, their cold serialized durations and their share of the step.

    python tools/launch_summary.py gpurun_out/launches_c2_r01.csv [steps] [warmup]

bench.py launches warm-up steps, the timed steps, then the end-to-end host-path calls;
the timed steps are evaluation launches warmup .. warmup + steps - 1 with their binning
kernels.
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    warmup = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    lines = open(path).read().splitlines()
    i = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[i:]))
    hdr = rows[0]
    ki, mi, vi, ii, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        per[int(r[ii])][r[mi]] = v
        nm = r[ki].split("(")[0]
        nm = nm[5:] if nm.startswith("void ") else nm
        names[int(r[ii])] = nm
    # our kernels only (sg_*); the last `steps` evaluation launches and everything between
    ours = [k for k in sorted(per) if names[k].startswith("sg_")]
    evals = [k for k in ours if names[k] == "sg_eval_kernel"]
    # timed region: the `steps` evaluation launches after warm-up, with their binning kernels
    sel = []
    if len(evals) >= warmup + steps:
        prev_eval = evals[warmup - 1] if warmup > 0 else -1
        sel = [k for k in ours if prev_eval < k <= evals[warmup + steps - 1]]
    agg = collections.OrderedDict()
    for k in sel:
        a = agg.setdefault(names[k], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += per[k].get("gpu__time_duration.sum", 0.0)
        a[2] += per[k].get("dram__bytes_read.sum", 0.0) + per[k].get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"{path}: {steps} timed steps, {len(sel)} launches of our kernels "
          f"({len(sel) / max(steps, 1):.0f} per step), {tot / max(steps, 1):.1f} us/step (ncu: cold, serialized)")
    for nm, (cnt, t, b) in agg.items():
        print(f"  {nm:28s} x{cnt / steps:.0f}/step  {t / cnt:10.1f} us/launch  {t / tot:6.1%} of step"
              + (f"  {b / cnt / 1e6:9.1f} MB DRAM/launch" if b else ""))


if __name__ == "__main__":
    main()
