"""Key metrics of an ncu --set full report (read here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
]
STALL = "smsp__average_warp_latency_issue_stalled_"
STALL2 = "smsp__pcsamp_warps_issue_stalled_"


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    recs = []
    for r in rows[2:]:
        recs.append({h: (v, u) for h, v, u in zip(hdr, r, units)})
    return recs


def table(paths):
    """Side-by-side key metrics of several single-kernel reports (knob pairs)."""
    import os
    recs = [raw(p)[0] for p in paths]
    names = [os.path.basename(p).replace(".ncu-rep", "")[-24:] for p in paths]
    print(f"{'metric':64s}" + "".join(f"{n:>26s}" for n in names))
    for k in KEYS:
        if all(k in r for r in recs):
            print(f"{k[:64]:64s}" + "".join(f"{r[k][0]:>26s}" for r in recs))
    for r, n in zip(recs, names):
        tot = sum(float(v.replace(',', '')) for k, (v, u) in r.items()
                  if k.startswith(STALL2) and v not in ('', 'n/a') and not k.endswith("_not_issued"))
        st = sorted(((float(v.replace(',', '')) if v not in ('', 'n/a') else 0.0, k)
                     for k, (v, u) in r.items() if k.startswith(STALL2)
                     and not k.endswith("_not_issued")), reverse=True)[:6]
        print(f"stalls {n}: " + ", ".join(f"{k[len(STALL2):]}={v / max(tot, 1):.0%}" for v, k in st))


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--table":
        return table(sys.argv[2:])
    for path in sys.argv[1:]:
        for rec in raw(path):
            print(f"== {path}  {rec.get('Kernel Name', ('?',))[0][:40]}")
            for k in KEYS:
                if k in rec:
                    v, u = rec[k]
                    print(f"  {k:70s} {v:>16s} {u}")
            st = sorted(((float(v.replace(',', '')) if v not in ('', 'n/a') else 0.0, k)
                         for k, (v, u) in rec.items() if k.startswith(STALL2)
                         and not k.endswith("_not_issued")), reverse=True)[:8]
            if st:
                tot = sum(float(v.replace(',', '')) for k, (v, u) in rec.items()
                          if k.startswith(STALL2) and v not in ('', 'n/a') and not k.endswith("_not_issued"))
                print("  top stall samples:", ", ".join(f"{k[len(STALL2):]}={v / max(tot, 1):.0%}" for v, k in st))


if __name__ == "__main__":
    main()
