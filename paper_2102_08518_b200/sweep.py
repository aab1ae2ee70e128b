"""(m, d) x branch-mode sweep harness with a CUDA backend.

Mirrors the reference harness (pkg/src/splinegen/bench.py:82-215): `run_sweep`
generates one kernel per lower-diagonal (group size m, pipeline depth d) cell
and branch mode, times its evaluation kernel with CUDA events (device time per batch), optionally hands each cell's outputs to a caller-supplied
checker (the tests pass one backed by the CPU oracle; the product never imports
it), and returns
`BenchRecord`s that `emit_csv` / `emit_matrix` write in the reference's formats
(CSV header `spline,m,d,branch_mode,backend,trials,mean_recon_per_sec,variance`,
gnuplot lower-diagonal matrices).  The timing is per batch as in the reference
(`_time_cell`, bench.py:152-165) but each batch is one device launch measured
with CUDA events, so mean/variance are over batches of `batch_size` queries.
"""

from __future__ import annotations

import io
from dataclasses import dataclass

import numpy as np

from . import runtime
from .api import DataVolume, Evaluator, sample_points
from .cudagen import GenConfig
from .schedule import BRANCH_MODES, ScheduleParams

CSV_HEADER = "spline,m,d,branch_mode,backend,trials,mean_recon_per_sec,variance"
CUDA = "cuda"


@dataclass(frozen=True)
class BenchRecord:
    spline: str
    m: int
    d: int
    branch_mode: str
    backend: str
    trials: int
    mean_recon_per_sec: float
    variance: float


def default_grid(n: int):
    return [(m, d) for m in range(1, n + 1) for d in range(m, n + 1)]


def run_sweep(space, data: DataVolume, grid=None, modes=BRANCH_MODES, trials: int = 1 << 20,
              seed: int = 0, batch_size: int = 1 << 18, refetch_tables: bool = False,
              unroll_cosets: bool = True, float_width: str = "f32", backend: str = CUDA,
              check=None, check_points: int = 32, **variant):
    """Time every (m, d, mode) cell on the GPU; one BenchRecord per cell.

    `check(pts, got, cell)`: optional verifier called with `check_points` query
    points (f64, (k, s)) and the cell's outputs for them (f64 numpy) -- the reference
    harness spot-checks against its oracle here (bench.py:126-136)."""
    import torch
    if backend != CUDA:
        raise ValueError(f"unknown backend {backend!r} (this package times the cuda backend)")
    n = space.stencil_size
    grid = default_grid(n) if grid is None else grid
    for m, d in grid:
        if d < m:
            raise ValueError(f"grid cell ({m}, {d}) violates depth >= group size")
    pts = sample_points(space, data, min(trials, batch_size), seed)
    dt = torch.float32 if float_width == "f32" else torch.float64
    xs = torch.from_numpy(pts).to(dt).cuda()
    tol = 1e-9 if float_width == "f64" else 1e-5
    records = []
    for m, d in sorted(grid):
        for mode in modes:
            cfg = GenConfig(params=ScheduleParams(m, d, mode, refetch_tables),
                            float_width=float_width, unroll_cosets=unroll_cosets, **variant)
            ev = Evaluator(space, data, cfg)
            ev(xs[: min(len(xs), 64)])                 # warm-up
            rates = []
            remaining = trials
            out = torch.empty(len(xs), dtype=dt, device=xs.device)
            grad = torch.empty_like(xs) if ev.prog.has_grad else None
            while remaining > 0:
                size = min(remaining, len(xs))
                # device time of the evaluation kernel alone (CUDA events on the launch
                # stream around the launch, inside the C ABI), not the Python call
                ev.module.kernel_time()
                ev.module.set_timing(True)
                runtime.eval_device(ev.module, ev.volume, xs[:size], out, grad)
                ev.module.set_timing(False)
                ms, _ = ev.module.kernel_time()
                rates.append(size / max(ms / 1e3, 1e-12))
                remaining -= size
            ev.module.status()
            if check is not None:
                p = pts[:check_points]
                got = ev(torch.from_numpy(p).to(dt).cuda())
                got = (got[0] if isinstance(got, tuple) else got).double().cpu().numpy()
                check(p, got, (m, d, mode, tol))
            arr = np.array(rates)
            records.append(BenchRecord(space.name, m, d, mode, backend, trials,
                                       float(arr.mean()), float(arr.var())))
    return records


def emit_csv(records) -> str:
    lines = [CSV_HEADER]
    for r in sorted(records, key=lambda r: (r.m, r.d, r.branch_mode, r.backend)):
        lines.append(f"{r.spline},{r.m},{r.d},{r.branch_mode},{r.backend},{r.trials},"
                     f"{r.mean_recon_per_sec!r},{r.variance!r}")
    return "\n".join(lines) + "\n"


def parse_csv(text: str):
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or lines[0] != CSV_HEADER:
        raise ValueError("missing or malformed CSV header")
    out = []
    for ln in lines[1:]:
        spline, m, d, mode, backend, trials, mean, var = ln.split(",")
        out.append(BenchRecord(spline, int(m), int(d), mode, backend, int(trials), float(mean),
                               float(var)))
    return out


def emit_matrix(records, branch_mode: str, field: str = "mean_recon_per_sec") -> str:
    cells = {(r.m, r.d): getattr(r, field) for r in records if r.branch_mode == branch_mode}
    if not cells:
        return ""
    mmax = max(m for m, _ in cells)
    dmax = max(d for _, d in cells)
    buf = io.StringIO()
    for d in range(1, dmax + 1):
        row = [("" if cells.get((m, d)) is None else repr(cells[(m, d)])) for m in range(1, mmax + 1)]
        buf.write("\t".join(row).rstrip("\t") + "\n")
    return buf.getvalue()
