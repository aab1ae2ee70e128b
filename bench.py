"""Benchmark of the hot path: batched spline reconstruction on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One JSON line on rank 0 (contract in the task statement).  A "step" is one
evaluation of the configuration's full query batch (one kernel launch over
N queries against a device-resident coset volume).  `value` is the whole-job
reconstruction rate in G reconstructions/s (queries of all ranks / max-over-
ranks device time); `e2e` is the same metric through the reference-facing C-ABI
host call (`sg_eval_host`: H2D of the queries from pinned memory, kernel, D2H
of the results, every step).

Configs (BASELINE.json, restated concretely in SURVEY.md 8d):
  c1   tricubic B-spline on Z^3, 64^3, 2^20 uniform queries
  c2   BCC quintic box spline, 2 x 101^3 coset-split, 2^24 uniform queries
  c3   BCC Voronoi spline (order 3), 2 x 203^3, 2^26 ray-ordered queries
  c4   FCC 6-direction box spline, 4 x 161^3, 2^26 uniform queries, value + gradient
  c4v  FCC Voronoi spline (order 3), 4 x 161^3, 2^26 uniform queries, value + gradient
  c4v4 FCC Voronoi spline (order 4, "cubic"), 4 x 161^3, 2^26 uniform, value + gradient
  c5   BCC Voronoi spline (order 3), 2 x 406^3, 2^30 ray-ordered queries, strong-scaled over
       the GPUs (default: the largest single-GPU configuration)
  c5u  c5 with uniform queries; c3r / c3rs the fused renderer of c3 (without / with shading);
  c3o2 / c4vo2 / c5o2 the order-2 Voronoi versions measured in round 1
Under torchrun every rank evaluates its own batch (weak scaling, volume replicated).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PROFILES = ROOT / "profiles"

# name -> workload (BASELINE.json configs, restated concretely in SURVEY.md 8d)
CONFIGS = {
    "c1": dict(space="tricubic", extents=(64, 64, 64), queries=1 << 20, kind="uniform",
               grad=False, scaling="weak", variant=dict(mode="binned", form="sym"),
               desc="tensor-product tricubic B-spline on Z^3, 64^3, 2^20 uniform"),
    "c1l": dict(space="tricubic", extents=(64, 64, 64), queries=1 << 20, kind="uniform",
                grad=False, scaling="weak", variant=dict(mode="direct", fetch="linear", block=256),
                desc="c1 through the hardware linear-fetch variant (SURVEY 8f row f4: 8 filtered "
                     "texture fetches instead of 64 reads; opt-in, ~3e-3 accurate, not the 1e-5 bar)"),
    "c2": dict(space="bcc_box5", extents=(101, 101, 101), queries=1 << 24, kind="uniform",
               grad=False, scaling="weak",
               variant=dict(mode="binned", coeffs="imm", form="sym", block=512),
               desc="BCC quintic box spline (4 dirs x2), 2x101^3 coset-split, 2^24 uniform"),
    "c3": dict(space="bcc_voronoi3", extents=(203, 203, 203), queries=1 << 26, kind="rays",
               rays=(512, 512, 256), grad=False, scaling="weak",
               variant=dict(mode="sorted", coeffs="imm", block=640, tile=3200, radix=1, min_blocks=1,
                            cmajor=3),
               desc="BCC Voronoi spline (order 3: the paper's BCC Voronoi case, 14 reference "
                    "polynomials), 2x203^3, 2^26 ray-ordered"),
    "c3o2": dict(space="bcc_voronoi2", extents=(203, 203, 203), queries=1 << 26, kind="rays",
                 rays=(512, 512, 256), grad=False, scaling="weak",
                 variant=dict(mode="sorted", coeffs="imm", block=512, radix=1),
                 desc="BCC Voronoi spline (order 2, piecewise cubic), 2x203^3, 2^26 ray-ordered"),
    "c4": dict(space="fcc_box6", extents=(161, 161, 161), queries=1 << 26, kind="uniform",
               grad=True, scaling="weak", variant=dict(mode="direct", coeffs="imm", block=128),
               desc="FCC 6-direction box spline, 4x161^3, 2^26 uniform, value + gradient"),
    "c4vo2": dict(space="fcc_voronoi2", extents=(161, 161, 161), queries=1 << 26, kind="uniform",
                grad=True, scaling="weak", variant=dict(mode="direct", coeffs="table", block=128),
                desc="FCC Voronoi spline (order 2), 4x161^3, 2^26 uniform, value + gradient"),
    "c4v": dict(space="fcc_voronoi3", extents=(161, 161, 161), queries=1 << 26, kind="uniform",
                 grad=True, scaling="weak",
                 variant=dict(mode="sorted", coeffs="imm", form="sym", block=640, tile=1280, min_blocks=1,
                              radix=1, presort=64, qhoist=1),
                 desc="FCC Voronoi spline (order 3, the paper's FCC case), 4x161^3, 2^26 uniform, "
                      "value + gradient"),
    "c4v4": dict(space="fcc_voronoi4", extents=(161, 161, 161), queries=1 << 26, kind="uniform",
                 grad=True, scaling="weak",
                 variant=dict(mode="sorted", coeffs="table", tloop=1, tchunk=112, block=384, radix=1,
                              presort=32, qhoist=1),
                 desc="FCC Voronoi spline (order 4, 'cubic'), 4x161^3, 2^26 uniform, value + gradient"),
    "c5u": dict(space="bcc_voronoi3", extents=(406, 406, 406), queries=1 << 30, kind="uniform",
                grad=False, scaling="strong", steps=20,
                variant=dict(mode="sorted", coeffs="imm", block=640, tile=3200, radix=1, min_blocks=1,
                             cmajor=3, presort=64),
                desc="c5 with uniform random queries (SURVEY 8d secondary): 535 MB volume > L2; "
                     "a locality pre-sort of the queries (64-cell bins) keeps the gathers in L2"),
    "c3r": dict(space="bcc_voronoi3", extents=(203, 203, 203), queries=1 << 26, kind="render",
                rays=(512, 512, 256), grad=False, scaling="weak", variant=dict(),
                desc="fused volume render of c3: 512x512 rays x 256 samples through 2x203^3 BCC "
                     "Voronoi (ray march + psi-sorted reconstruction + compositing in one kernel)"),
    "c3rs": dict(space="bcc_voronoi3", extents=(203, 203, 203), queries=1 << 26, kind="render",
                 rays=(512, 512, 256), grad=True, scaling="weak", variant=dict(),
                 desc="c3r with gradient (Lambert) shading at every sample"),
    "c5": dict(space="bcc_voronoi3", extents=(406, 406, 406), queries=1 << 30, kind="rays",
               rays=(1024, 1024, 1024), grad=False, scaling="strong", steps=20,
               variant=dict(mode="sorted", coeffs="imm", block=640, tile=3200, radix=1, min_blocks=1,
                            cmajor=3),
               desc="BCC Voronoi spline (order 3), 2x406^3, 2^30 ray-ordered sharded over the GPUs"),
    "c5o2": dict(space="bcc_voronoi2", extents=(406, 406, 406), queries=1 << 30, kind="rays",
                 rays=(1024, 1024, 1024), grad=False, scaling="strong", steps=20,
                 variant=dict(mode="sorted", coeffs="imm", block=512, radix=1),
                 desc="BCC Voronoi spline (order 2), 2x406^3, 2^30 ray-ordered sharded over the GPUs"),
}
DEFAULT_CONFIG = "c5"


def _space_available(name):
    from paper_2102_08518_b200.model import SPACES_DIR
    return (SPACES_DIR / f"{name}.json").exists()


def default_config_name():
    return DEFAULT_CONFIG if _space_available(CONFIGS[DEFAULT_CONFIG]["space"]) else "c1"


def gen_config_for(space, grad=False, **over):
    """The tuned default variant per space (see profiles/ for the variant sweeps)."""
    from paper_2102_08518_b200 import GenConfig, ScheduleParams
    n = space.stencil_size
    kw = dict(params=ScheduleParams(1, n, "predicated"), float_width="f32",
              unroll_cosets=True, form="horner", block=256, grad=grad,
              mode="binned", coeffs="table" if space.nref > 2 else "imm")
    kw.update(over)
    return GenConfig(**kw)


def build_program(cfg_name, **over):
    """The configuration's measured-best variant (CONFIGS[..]['variant']), plus overrides."""
    from paper_2102_08518_b200 import generate, load_fixture
    c = CONFIGS[cfg_name]
    space = load_fixture(c["space"])
    kw = dict(c.get("variant", {}))
    kw.update(over)
    return space, generate(space, gen_config_for(space, c["grad"], **kw), c["extents"])


def precompile_bench_kernels():
    from paper_2102_08518_b200.runtime import compile_source
    for name, c in CONFIGS.items():
        if not _space_available(c["space"]):
            continue
        if c["kind"] == "render":
            from paper_2102_08518_b200 import generate, load_fixture
            from paper_2102_08518_b200.render import render_config
            space = load_fixture(c["space"])
            prog = generate(space, render_config(space, c["grad"], **c.get("variant", {})),
                            c["extents"])
        else:
            _, prog = build_program(name)
        compile_source(prog.source)


def falg_per_query(space_name, grad=False):
    """Reference dynamic FP-op count (m=1, d=n, branchy), pinned by the golden script; with
    `grad`, plus the gradient's ops by the same counting rule applied to the reference's
    derivative polynomials (tests/golden/make_golden.py: falg_gradient_extra)."""
    p = ROOT / "tests" / "golden" / "falg.json"
    d = json.loads(p.read_text()) if p.exists() else {}
    return d.get(space_name + "+grad" if grad else space_name)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    d = json.loads(p.read_text()) if p.exists() else {}
    sm_mhz = d.get("sm_max_mhz", 1965.0)
    fp32 = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12   # TFLOP/s: SMs x FP32 lanes x FMA x clock
    return dict(fp32_tflops=fp32, hbm_gbs=d.get("hbm_gbs", 6650.0), sm_max_mhz=sm_mhz,
                source="MEASURED_PEAKS.json" if p.exists() else "fallback")


# -- clocks ---------------------------------------------------------------------------


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:   # sampler is live before timing
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# -- CPU baseline (oracle port; test-infrastructure import, baseline leg only) ---------------


_CPU_STATE = {}


def _cpu_worker(i):
    """Evaluate shard i of the sample (state inherited copy-on-write through fork)."""
    from oracle import refeval
    st = _CPU_STATE
    sp = refeval.load_space_file(st["path"])
    xs = st["xs"][i * st["shard"]:(i + 1) * st["shard"]].astype(np.float64)
    t0 = time.perf_counter()
    refeval.reference_eval_batch(sp, xs, st["arrays"])
    return time.perf_counter() - t0


def cpu_baseline(space_name, arrays_f32, xs_f32, budget_s=15.0, shard=1 << 14, pool=None):
    """Time the oracle port (restatement of reference_eval_batch, numpy f64) on all
    host cores over a bounded sample of the same workload."""
    import multiprocessing as mp
    from paper_2102_08518_b200.model import SPACES_DIR
    path = str(SPACES_DIR / f"{space_name}.json")
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    if _CPU_STATE.get("path") != path or _CPU_STATE.get("xs") is not xs_f32:
        _CPU_STATE.update(path=path, arrays=[a.astype(np.float64) for a in arrays_f32],
                          xs=xs_f32, shard=shard, rate1=None)
    cores = len(os.sched_getaffinity(0))
    if _CPU_STATE.get("rate1") is None:
        t1 = _cpu_worker(0)     # calibrate on one shard
        _CPU_STATE["rate1"] = shard / t1
    rate1 = _CPU_STATE["rate1"]
    nshards = max(cores, int(budget_s * rate1 * cores / shard) // cores * cores)
    nshards = min(nshards, max(1, len(xs_f32) // shard))
    own = pool is None
    if own:
        pool = mp.get_context("fork").Pool(cores)
    t0 = time.perf_counter()
    pool.map(_cpu_worker, range(nshards), chunksize=1)
    wall = time.perf_counter() - t0
    if own:
        pool.close()
        pool.join()
    n = nshards * shard
    return {"value": n / wall / 1e9, "unit": "Grecon/s", "cores": cores, "kind": "port",
            "cpu_model": cpu_model(), "rate_1core": rate1 / 1e9,
            "sample": f"{n} of the configuration's queries ({nshards} shards of {shard}), "
                      f"oracle/refeval.reference_eval_batch (numpy f64, restatement of "
                      f"splinegen.oracle.reference_eval_batch) on {cores} processes, "
                      f"{wall:.2f}s; 1-core rate {rate1:.3e} q/s"}


# -- workload ---------------------------------------------------------------------------


def query_range(cfg_name, rank, world):
    """This rank's slice of the global query stream (weak: n per rank; strong: shard)."""
    from paper_2102_08518_b200.dist import shard_range
    c = CONFIGS[cfg_name]
    if c["scaling"] == "strong":
        return shard_range(c["queries"], rank, world)
    return rank * c["queries"], (rank + 1) * c["queries"]


def make_queries(cfg_name, lo, hi, device, chunk=1 << 25):
    """Queries [lo, hi) of the configuration's global stream, generated in chunks on
    `device` (the generators use fp64 temporaries; chunking bounds their footprint)."""
    import torch
    from paper_2102_08518_b200 import queries
    c = CONFIGS[cfg_name]
    out = torch.empty((hi - lo, len(c["extents"])), dtype=torch.float32, device=device)
    for a in range(lo, hi, chunk):
        b = min(hi, a + chunk)
        if c["kind"] == "rays":
            w, h, st = c["rays"]
            total = w * h * st
            # weak-scaled ranks beyond the first replay the ray stream (same work per rank)
            a0 = a % total
            out[a - lo:b - lo] = queries.rays(a0, a0 + (b - a), c["extents"], w, h, st, 2, device)
        else:
            out[a - lo:b - lo] = queries.uniform(a, b, c["extents"], 1, device)
    return out


def make_inputs(cfg_name, rank, device, world=1):
    from paper_2102_08518_b200 import load_fixture
    c = CONFIGS[cfg_name]
    space = load_fixture(c["space"])
    ext = c["extents"]
    rng = np.random.default_rng(0)  # make_volume(seed=0): U[0,1), cosets in order
    arrays = [rng.random(ext).astype(np.float32) for _ in range(space.ncosets)]
    lo, hi = query_range(cfg_name, rank, world)
    xs = make_queries(cfg_name, lo, hi, device)
    return space, arrays, xs


def config_dict(cfg_name, world):
    """The line's `config` object -- built identically by both arms (ours and --impl
    reference), so the driver can match them."""
    from paper_2102_08518_b200 import load_fixture
    c = CONFIGS[cfg_name]
    sp = load_fixture(c["space"])
    lo, hi = query_range(cfg_name, 0, world)
    n = hi - lo
    d = {"workload": cfg_name + ": " + c["desc"], "space": c["space"],
         "extents": list(c["extents"]), "cosets": sp.ncosets, "query_kind": c["kind"]}
    if c["kind"] == "render":
        w, h, steps = c["rays"]
        d.update({"image": [w, h], "samples_per_ray": steps, "samples_per_gpu": w * h * steps,
                  "shading": c["grad"], "parallelism": f"full image per GPU x{world}",
                  "l2": "no query/result streams: samples are generated and consumed in registers"})
        return d
    d.update({"queries_per_gpu": n, "gradient": c["grad"],
              "parallelism": f"query shards x{world}, volume replicated",
              "l2": "L2 flushed between steps" if n * sp.dim * 4 < 2 * 126e6
              else "query stream > L2 (126 MB); volume L2-resident by design"
              if 4 * sp.ncosets * math.prod(c["extents"]) < 100e6
              else "query stream and volume > L2 (126 MB)"})
    return d


def cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def roofline(cfg_name, falg, n, eval_kernel_ms, step_ms, pk, kernel_key=None):
    """roofline block of the bench line for the dominant kernel (sg_eval_kernel).

    achieved = algorithmic FP32 work (the reference's own dynamic op count F_alg per query,
    SURVEY 8d) x queries / the kernel's CUDA-event time; peak = FP32 FMA peak.  The
    kernel may execute fewer flops than F_alg (symmetry-rewritten / factored forms), so
    `executed` restates the same time against the FP32 flops the kernel actually ran and
    `issue` against the SM issue rate (4 warp-instructions / clk / SM) -- both counted by
    ncu on the same launch (profiles/ncu_<config>.json)."""
    if not falg:
        return None
    from paper_2102_08518_b200 import load_fixture
    c = CONFIGS[cfg_name]
    sp = load_fixture(c["space"])
    # T_floor = max(F_alg / P_fp32, B_alg / BW), BW = HBM when the coset
    # volume exceeds L2.  B_alg = 4 B per coefficient gather (mean stencil size over the
    # sub-regions' polynomials) + the query and result streams (+ gradient)
    nbar = float(np.mean([len(sb.stencil) for sb in sp.subregions]))
    balg = 4 * nbar * sp.ncosets + 4 * sp.dim + 4 + (4 * sp.dim if c["grad"] else 0)
    vol_bytes = 4 * sp.ncosets * math.prod(c["extents"])
    t_fp = falg / (pk["fp32_tflops"] * 1e12)
    t_hbm = balg / (pk["hbm_gbs"] * 1e9)
    hbm_block = None
    if vol_bytes > 126e6 or t_hbm > t_fp:
        a = balg * n / (eval_kernel_ms / 1e3) / 1e9
        hbm_block = {"bytes_per_query": round(balg, 1), "achieved": round(a, 1),
                     "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": round(a / pk["hbm_gbs"], 4),
                     "volume_bytes": vol_bytes}
    achieved = falg * n / (eval_kernel_ms / 1e3) / 1e12
    if c["grad"]:
        f0 = falg_per_query(c["space"])
        a0 = f0 * n / (eval_kernel_ms / 1e3) / 1e12
        value_only = {"falg": f0, "achieved": round(a0, 3), "frac": round(a0 / pk["fp32_tflops"], 4),
                      "unit": "TFLOP/s", "note": "value-only F_alg (the reference evaluates no gradient)"}
    if hbm_block and t_hbm > t_fp:
        roof = {"bound": "hbm", "achieved": hbm_block["achieved"], "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": hbm_block["frac"], "traffic": None,
                "fp32": {"achieved": round(achieved, 3), "peak": round(pk["fp32_tflops"], 2),
                         "unit": "TFLOP/s", "frac": round(achieved / pk["fp32_tflops"], 4)}}
    else:
        roof = {"bound": "fp32", "achieved": round(achieved, 3), "peak": round(pk["fp32_tflops"], 2),
                "unit": "TFLOP/s", "frac": round(achieved / pk["fp32_tflops"], 4), "traffic": None}
        if hbm_block:
            roof["hbm"] = hbm_block
    if c["grad"]:
        roof["value_only"] = value_only
    roof.update({
            "note": f"F_alg = {falg:g} FP ops/query (reference dynamic count, m=1 d=n branchy"
                    + ("; value + gradient: the same counting rule on the derivative polynomials"
                       if c["grad"] else "") + f"; tests/golden/falg.json) x {n} queries / sg_eval_kernel time "
                    f"({eval_kernel_ms:.4f} ms of the {step_ms:.4f} ms step, CUDA events on the "
                    f"launch stream); peak = 148 SM x 128 FP32 lanes x 2 x {pk['sm_max_mhz']:.0f} MHz "
                    f"({pk['source']} sm_max_mhz); binding roof = max(F_alg / FP32 peak, "
                    f"B_alg / HBM) per query (SURVEY 8d)"})
    prof = PROFILES / f"ncu_{cfg_name}.json"
    d = json.loads(prof.read_text()) if prof.exists() else None
    if d is not None and d.get("kernel_key") != kernel_key:
        roof["profile"] = f"{prof.name} is from another kernel variant (stale): not used"
        d = None
    if d is not None:
        roof["traffic"] = d.get("dram_bytes_per_launch")
        ex = d.get("executed_fp32_flops_per_query")
        if ex:
            a = ex * n / (eval_kernel_ms / 1e3) / 1e12
            roof["executed"] = {"flops_per_query": round(ex, 1), "achieved": round(a, 3),
                                "frac": round(a / pk["fp32_tflops"], 4), "unit": "TFLOP/s"}
        wi = d.get("warp_inst_per_query")
        if wi:
            peak_gi = 148 * 4 * pk["sm_max_mhz"] / 1e3          # G warp-instructions / s
            a = wi * n / (eval_kernel_ms / 1e3) / 1e9
            roof["issue"] = {"warp_inst_per_query": round(wi, 2), "achieved": round(a, 1),
                             "peak": round(peak_gi, 1), "unit": "Gwarp-inst/s",
                             "frac": round(a / peak_gi, 4)}
        roof["profile"] = f"profiles/ncu_{cfg_name}.json ({d.get('source', '')})"
    l2p = PROFILES / "r01_l2_bandwidth.json"
    if l2p.exists():
        # the coefficient gathers against the measured L2 read bandwidth (algorithmic bytes:
        # one 4-B read per stencil site and coset)
        from paper_2102_08518_b200 import load_fixture
        c = CONFIGS[cfg_name]
        gbytes = 4 * nbar * sp.ncosets
        l2 = json.loads(l2p.read_text()).get("l2_gbs")
        if l2:
            a = gbytes * n / (eval_kernel_ms / 1e3) / 1e9
            roof["l2_gathers"] = {"bytes_per_query": round(gbytes, 1), "achieved": round(a, 1), "peak": l2,
                                  "unit": "GB/s", "frac": round(a / l2, 4),
                                  "peak_source": "profiles/r01_l2_bandwidth.json"}
    return roof


def run_ours(args, rank, world, device):
    import torch
    import torch.distributed as dist
    from paper_2102_08518_b200 import Evaluator
    from paper_2102_08518_b200 import runtime

    c = CONFIGS[args.config]
    space, arrays, xs = make_inputs(args.config, rank, device, world)
    _, prog = build_program(args.config)
    # volume: rank 0's synthetic data broadcast over NCCL (replicated per GPU)
    if world > 1:
        dev_arrays = [torch.from_numpy(a).to(device) for a in arrays]
        for t in dev_arrays:
            dist.broadcast(t, 0)
        ev = Evaluator(space, dev_arrays, prog=prog, device=device.index)
    else:
        ev = Evaluator(space, arrays, prog=prog, device=device.index)
    n = xs.shape[0]
    out = torch.empty(n, dtype=torch.float32, device=device)
    grad = torch.empty((n, space.dim), dtype=torch.float32, device=device) if prog.has_grad else None
    stream = torch.cuda.current_stream(device)
    l2_flush = None
    if n * space.dim * 4 < 2 * 126e6:
        l2_flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=device)

    def step():
        runtime.eval_device(ev.module, ev.volume, xs, out, grad, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(device)
    ev.module.status()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev.module.kernel_time()          # reset
    ev.module.set_timing(True)       # events around the evaluation kernel alone
    with ClockSampler(device.index) as clk:
        t_wall = time.perf_counter()
        for i in range(args.steps):
            if l2_flush is not None:
                l2_flush.fill_(float(i))
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize(device)
        t_wall = time.perf_counter() - t_wall
    if world > 1:
        dist.barrier()
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    ev.module.set_timing(False)
    kms, klaunches = ev.module.kernel_time()
    eval_kernel_ms = kms / max(1, klaunches)
    ev.module.status()
    # max over ranks
    tt = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    per_step_total = c["queries"] if c["scaling"] == "strong" else n * world
    total_q = per_step_total * args.steps
    value = total_q / (ms / 1e3) / 1e9
    kernel_ms = ms / args.steps

    gather_ms = None
    if args.gather and world > 1:
        # optional: every rank receives all ranks' results (reported beside, not inside, value)
        from paper_2102_08518_b200.dist import gather_results
        total = c["queries"] if c["scaling"] == "strong" else n * world
        gather_results(out, total, device=device)
        torch.cuda.synchronize(device)
        dist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        gather_results(out, total, device=device)
        g1.record(stream)
        torch.cuda.synchronize(device)
        gather_ms = float(torch.tensor([g0.elapsed_time(g1)], dtype=torch.float64, device=device).item())
        gt = torch.tensor([gather_ms], dtype=torch.float64, device=device)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gather_ms = float(gt.item())

    # ---- end to end through the C-ABI host path (pinned buffers)
    xs_host = xs.cpu().pin_memory()
    out_host = torch.empty(n, dtype=torch.float32).pin_memory()
    grad_host = torch.empty((n, space.dim), dtype=torch.float32).pin_memory() if grad is not None else None
    e2e_steps = max(3, min(args.steps, 20))
    lib = runtime.lib()

    # the library's default chunk (2^21 queries, at least 4 chunks down to 2^18): H2D, kernel
    # and D2H overlap on 3 streams; measured on B200 (tools/e2e_chunks.py, round 2): c2 4.17
    # G/s at 2^21 vs 3.96 at 2^22, c3 4.24 at 2^21, c1 (2^20 queries) 2.84 at 2^18 vs 2.57 at 2^20
    host_chunk = min(1 << 21, max(1 << 18, n // 4))   # the C ABI's default chunk rule

    def host_step():
        runtime._check(lib.sg_eval_host(ev.module.handle, ev.volume.handle,
                                        runtime.ctypes.c_void_p(xs_host.data_ptr()), n,
                                        runtime.ctypes.c_void_p(out_host.data_ptr()),
                                        runtime.ctypes.c_void_p(grad_host.data_ptr() if grad_host is not None else 0),
                                        host_chunk))
    host_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        host_step()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = per_step_total * e2e_steps / float(te.item()) / 1e9
    # correctness spot check of the timed kernel against the host path
    ref_out = out[:4096].cpu()
    assert torch.equal(ref_out, out_host[:4096]), "device and host paths disagree"

    if rank != 0:
        return None
    pk = peaks()
    falg = falg_per_query(c["space"], c["grad"])
    roof = roofline(args.config, falg, n, eval_kernel_ms, kernel_ms, pk, prog.key)
    line = {
        "metric": "G reconstructions/sec per B200 (fraction of FP32 roofline in roofline)",
        "value": round(value, 4), "unit": "Grecon/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(kernel_ms, 4), "higher_is_better": True,
        "scaling": c["scaling"], "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args.config, world),
        "e2e": {"value": round(e2e_value, 4), "unit": "Grecon/s",
                "h2d_bytes_per_step": n * space.dim * 4,
                "d2h_bytes_per_step": n * 4 * (1 + (space.dim if grad is not None else 0)),
                "steps": e2e_steps, "path": "sg_eval_host (C ABI, pinned host buffers, "
                f"H2D / kernel / D2H pipelined over {host_chunk}-query chunks on 3 streams)"},
        "gpu_launches": args.steps * (4 if prog.mode == "binned" else 1),
        "roofline": roof,
        "clocks": clk.summary(),
        "kernel": {"regs": ev.module.regs()[0], "fetch_mode": prog.meta["fetch_mode"],
                   "form": prog.config.form, "coeffs": prog.config.coeffs, "mode": prog.mode,
                   "bin": prog.bin, "brick": list(prog.brick), "block": prog.block,
                   "eval_kernel_ms": round(eval_kernel_ms, 4), "wall_s": round(t_wall, 3)},
        "gather_ms": gather_ms,
        "gpu_launches_note": "per step: query sort (sg_bin_count, sg_bin_plan, sg_bin_scatter_tiled) "
                             "+ sg_eval_kernel" if prog.mode == "binned" else "1 kernel per step",
    }
    if not args.no_cpu and world == 1:   # the CPU baseline is an N = 1 figure
        xs_np = xs[: 1 << 20].cpu().numpy()
        line["cpu_baseline"] = cpu_baseline(c["space"], arrays, xs_np, budget_s=args.cpu_budget,
                                            shard=1 << 12)
    return line


def run_render(args, rank, world, device):
    """Fused renderer configs: one step = one image."""
    import torch
    from paper_2102_08518_b200 import load_fixture
    from paper_2102_08518_b200.render import Renderer
    c = CONFIGS[args.config]
    space = load_fixture(c["space"])
    rng = np.random.default_rng(0)
    arrays = [rng.random(c["extents"]).astype(np.float32) for _ in range(space.ncosets)]
    w, h, steps = c["rays"]
    r = Renderer(space, arrays, w, h, steps, shade=c["grad"], device=device.index, **c.get("variant", {}))
    stream = torch.cuda.current_stream(device)
    for _ in range(args.warmup):
        r.launch(stream)
    torch.cuda.synchronize(device)
    r.ev.module.status()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device.index) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            r.launch(stream)
        e1.record(stream)
        torch.cuda.synchronize(device)
    ms = e0.elapsed_time(e1)
    tt = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    n = r.samples
    value = n * world * args.steps / (ms / 1e3) / 1e9
    step_ms = ms / args.steps
    # end to end: rays from pinned host memory, render, image back to the host, every step
    from paper_2102_08518_b200 import runtime
    rays_h = torch.from_numpy(r.rays_np).pin_memory()
    img_h = torch.empty((w * h, 4), dtype=torch.float32).pin_memory()
    e2e_steps = max(3, min(args.steps, 20))
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        r.rays.copy_(rays_h, non_blocking=True)
        r.launch(stream)
        img_h.copy_(r.rgba, non_blocking=True)
        torch.cuda.synchronize(device)
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = n * world * e2e_steps / float(te.item()) / 1e9
    r.ev.module.status()
    if rank != 0:
        return None
    pk = peaks()
    falg = falg_per_query(c["space"], c["grad"])
    roof = roofline(args.config, falg, n, step_ms, step_ms, pk, r.prog.key)
    line = {
        "metric": "G reconstructions/sec per B200 (fraction of FP32 roofline in roofline)",
        "value": round(value, 4), "unit": "Grecon/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True,
        "scaling": c["scaling"], "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args.config, world),
        "e2e": {"value": round(e2e_value, 4), "unit": "Grecon/s",
                "h2d_bytes_per_step": int(r.rays_np.nbytes), "d2h_bytes_per_step": w * h * 16,
                "steps": e2e_steps, "path": "ray table H2D (pinned), sg_render, rgba D2H"},
        "gpu_launches": args.steps,
        "roofline": roof,
        "clocks": clk.summary(),
        "kernel": {"regs": r.ev.module.regs()[0], "mode": "render", "block": r.prog.block},
    }
    if not args.no_cpu and world == 1:
        from oracle import refeval
        from oracle import render as orender
        from paper_2102_08518_b200.model import SPACES_DIR
        osp = refeval.load_space_file(SPACES_DIR / f"{c['space']}.json")
        npx = 64
        t0 = time.perf_counter()
        orender.render(osp, arrays, r.rays_np[:npx], steps, r.tf_np, shade=c["grad"])
        dt = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": npx * steps / dt / 1e9, "unit": "Grecon/s", "cores": 1,
                                "kind": "port",
                                "sample": f"{npx} rays x {steps} samples through oracle/render.py "
                                          f"(numpy f64 restatement of the reference evaluator + "
                                          f"compositing), 1 process, {dt:.2f}s"}
    return line


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU evaluator (oracle port) on all host cores,
    each step a bounded sample of the configuration's query stream."""
    if rank != 0:
        return None
    import multiprocessing as mp
    from paper_2102_08518_b200 import load_fixture
    c = CONFIGS[args.config]
    space = load_fixture(c["space"])
    rng = np.random.default_rng(0)
    arrays = [rng.random(c["extents"]).astype(np.float32) for _ in range(space.ncosets)]
    if c["kind"] == "render":
        return run_reference_render(args, c, space, arrays)
    # the fixed 2^20-query prefix of the configuration's stream, generated by
    # the same index-addressable generator the GPU arm uses
    xs = make_queries(args.config, 0, 1 << 20, "cpu").numpy()
    total_budget = 10.0 * args.cpu_budget       # seconds for the whole run (default 150 s)
    per_step = total_budget / (args.steps + args.warmup)
    cores = len(os.sched_getaffinity(0))
    shard = 1 << 11
    _cpu_worker_init(args.config, arrays, xs, shard)
    pool = mp.get_context("fork").Pool(cores)
    vals = []
    try:
        for i in range(args.warmup + args.steps):
            r = cpu_baseline(c["space"], arrays, xs, budget_s=per_step, shard=shard, pool=pool)
            if i >= args.warmup:
                vals.append(r)
    finally:
        pool.close()
        pool.join()
    v = statistics.median([r["value"] for r in vals])
    return {
        "impl": "reference",
        "metric": "G reconstructions/sec per B200 (fraction of FP32 roofline in roofline)",
        "value": v, "unit": "Grecon/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": None, "higher_is_better": True, "scaling": c["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config, world),
        "cpu_baseline": {**vals[-1], "value": v},
        "e2e": {"value": v, "unit": "Grecon/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_reference_render(args, c, space, arrays):
    """--impl reference for the renderer configs: the oracle renderer (reference evaluator
    restatement + compositing) on a bounded number of rays per step, one process."""
    from oracle import refeval
    from oracle import render as orender
    from paper_2102_08518_b200.model import SPACES_DIR
    from paper_2102_08518_b200.queries import ray_table
    from paper_2102_08518_b200.render import DEFAULT_TF, tf_vector
    w, h, steps = c["rays"]
    rays = ray_table(c["extents"], w, h, steps)
    tf = tf_vector(**DEFAULT_TF)
    osp = refeval.load_space_file(SPACES_DIR / f"{c['space']}.json")
    arr = [a.astype(np.float64) for a in arrays]
    npx = 32
    vals = []
    for i in range(args.warmup + args.steps):
        sl = rays[(i * npx) % len(rays):(i * npx) % len(rays) + npx]
        t0 = time.perf_counter()
        orender.render(osp, arr, sl, steps, tf, shade=c["grad"])
        if i >= args.warmup:
            vals.append(len(sl) * steps / (time.perf_counter() - t0) / 1e9)
    v = statistics.median(vals)
    return {"impl": "reference", "metric": "G reconstructions/sec per B200 (fraction of FP32 roofline in roofline)",
            "value": v, "unit": "Grecon/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": c["scaling"], "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, 1),
            "cpu_baseline": {"value": v, "unit": "Grecon/s", "cores": 1, "kind": "port",
                             "cpu_model": cpu_model(),
                             "sample": f"{npx} rays x {steps} samples per step, oracle/render.py"},
            "e2e": {"value": v, "unit": "Grecon/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def _cpu_worker_init(cfg_name, arrays, xs, shard):
    from paper_2102_08518_b200.model import SPACES_DIR
    _CPU_STATE.update(path=str(SPACES_DIR / f"{CONFIGS[cfg_name]['space']}.json"),
                      arrays=[a.astype(np.float64) for a in arrays], xs=xs, shard=shard, rate1=None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default: the configuration's, 300 or 20 for c5)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=None)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--gather", action="store_true",
                    help="also time the optional result gather to every rank (all_gather over "
                         "NCCL/NVLink, SURVEY 8e), reported separately as gather_ms")
    args = ap.parse_args()
    args.config = args.config or default_config_name()
    if args.steps is None:
        args.steps = CONFIGS[args.config].get("steps", 300)
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
        if line:
            print(json.dumps(line), flush=True)
        return 0
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SPLINEGPU_DIST_BACKEND=gloo lets several ranks share one GPU (code-path checks of the
    # multi-rank bench on a 1-GPU box); production runs use NCCL, one rank per GPU
    backend = os.environ.get("SPLINEGPU_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= max(1, torch.cuda.device_count())
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    if CONFIGS[args.config]["kind"] == "render":
        line = run_render(args, rank, world, device)
    else:
        line = run_ours(args, rank, world, device)
    if line:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
