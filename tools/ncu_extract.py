"""Summarise an ncu --set full capture of a bench configuration's evaluation kernel
into profiles/ncu_<config>.json (read by bench.py for roofline.traffic / .executed / .issue).

    python tools/ncu_extract.py <config> gpurun_out/prof_<config>.ncu-rep [tag]
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from tools.ncu_summary import raw  # noqa: E402


def num(rec, k):
    v = rec.get(k, ("0", ""))[0].replace(",", "")
    try:
        return float(v)
    except ValueError:
        return 0.0


def kernel_key(cfg):
    """Source hash of the configuration's kernel (bench.py ignores a stale profile)."""
    c = bench.CONFIGS[cfg]
    if c["kind"] == "render":
        from paper_2102_08518_b200 import generate, load_fixture
        from paper_2102_08518_b200.render import render_config
        sp = load_fixture(c["space"])
        return generate(sp, render_config(sp, c["grad"], **c.get("variant", {})), c["extents"]).key
    return bench.build_program(cfg)[1].key


def main():
    cfg, rep = sys.argv[1], sys.argv[2]
    tag = sys.argv[3] if len(sys.argv) > 3 else "r01"
    recs = [r for r in raw(rep) if "sg_eval_kernel" in r.get("Kernel Name", ("",))[0]]
    rec = recs[-1]
    c = bench.CONFIGS[cfg]
    n = c["queries"] if c["scaling"] != "strong" else c["queries"]
    unit = rec.get("gpu__time_duration.sum", ("", ""))[1]
    t = num(rec, "gpu__time_duration.sum")
    t_ms = t * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                "msecond": 1.0}.get(unit, 1.0)
    def nbytes(k):
        v = num(rec, k)
        u = rec.get(k, ("", ""))[1]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    # the full set carries per-cycle rates (summed over SMSPs); x elapsed cycles = counts
    cyc = num(rec, "smsp__cycles_elapsed.avg")
    ffma2 = num(rec, "derived__smsp__sass_thread_inst_executed_op_ffma_pred_on_x2") * cyc
    fadd = num(rec, "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum.per_cycle_elapsed") * cyc
    fmul = num(rec, "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum.per_cycle_elapsed") * cyc
    out = {
        "config": cfg, "tag": tag, "kernel": "sg_eval_kernel", "queries_per_launch": n,
        "source": f"ncu --set full --clock-control none (one launch of bench.py --config {cfg})",
        "ncu_kernel_ms": round(t_ms, 4),
        "dram_bytes_per_launch": nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum"),
        "warp_inst_per_query": num(rec, "smsp__inst_executed.sum") / n,
        "executed_fp32_flops_per_query": (ffma2 + fadd + fmul) / n,
        "issue_active_pct": num(rec, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": num(rec, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "alu_pipe_pct": num(rec, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "l1tex_throughput_pct": num(rec, "l1tex__throughput.avg.pct_of_peak_sustained_active"),
        "l1_hit_pct": num(rec, "l1tex__t_sector_hit_rate.pct"),
        "l2_hit_pct": num(rec, "lts__t_sector_hit_rate.pct"),
        "warps_active_pct": num(rec, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": num(rec, "launch__registers_per_thread"),
        "kernel_key": kernel_key(cfg),
    }
    p = ROOT / "profiles" / f"ncu_{cfg}.json"
    p.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
