"""Generate the golden vectors that pin the oracle (and through it the CUDA path).

Runs the UNMODIFIED reference package (`splinegen`, imported read-only from
/root/reference/pkg/src in the build container) on seeded inputs and writes:

  tests/golden/spaces/<name>.json   the space description the vectors were made on
                                    (reference fixtures are re-serialized with the
                                    reference's own `serialize_space`)
  tests/golden/<name>.npz           inputs (fp32 volumes + fp32 queries) and the
                                    reference outputs: reference_eval_batch values,
                                    per-coset lattice shift k and sub-region index
                                    (oracle._rho / oracle._membership), and
                                    interpret_batch results of f64/f32 programs
  tests/golden/falg.json            the reference's dynamic FP-op count per query of
                                    the canonical program (m=1, d=n, branchy),
                                    bench.py's algorithmic-FLOP figure

Usage (build container only; /root/reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [extra_space.json ...]

Extra spaces (our Part-I producer's output, paper_2102_08518_b200/spaces/*.json)
are parsed AND validated by the reference's own `parse_space`, so every space
the GPU path is parity-tested on is one the reference accepts.
"""

from __future__ import annotations

import json
import os
import sys
from collections import Counter
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path(os.environ.get("SPLINEGEN_REF", "/root/reference/pkg/src"))
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))

from splinegen import oracle as ref_oracle  # noqa: E402
from splinegen.bench import make_volume, sample_points  # noqa: E402
from splinegen.codegen import GenConfig, generate  # noqa: E402
from splinegen.ir import DataVolume, interpret_batch  # noqa: E402
from splinegen.model import fixture_text, parse_space, serialize_space  # noqa: E402
from splinegen.schedule import ScheduleParams  # noqa: E402

FIXTURES = {
    "linear1d": (16,),
    "halfgrid1d": (16,),
    "zp": (8, 8),
    "zp_k2": (8, 8),
    "trilinear": (6, 6, 6),
    "trilinear_voronoi": (6, 6, 6),
}

FP_OPS = ("fadd", "fsub", "fmul", "fneg", "fdiv")


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def adversarial_points(space, extents, rng, count):
    """Inputs that expose fp32 selection bugs: k+1/2 +- 1 ulp(f32),
    tiny |x| next to coset offsets, points exactly on BSP planes (>= decides),
    and points outside [0, E) (periodic wrap)."""
    s = space.dim
    e = np.array(extents, dtype=np.float64)
    pts = []
    per = max(1, count // 5)
    # 1) k + 1/2 (+-1 ulp f32) on random axes
    base = np.floor(rng.random((per, s)) * e) + 0.5
    for sign in (-1, 0, 1):
        p = base.astype(np.float32)
        if sign:
            p = np.nextafter(p, np.float32(sign * np.inf))
        pts.append(p.astype(np.float64))
    # 2) tiny coordinates next to coset offsets
    tiny = (rng.random((per, s)) - 0.5) * 2e-9
    for off in space.lattice.cosets:
        o = np.array([float(q) for q in off])
        pts.append(_f32(o + tiny + np.floor(rng.random((per, s)) * 2)))
    # 3) exactly on BSP planes, at dyadic positions near lattice sites
    if space.planes:
        for plane in space.planes:
            nrm = np.array([float(v) for v in plane.normal])
            site = np.floor(rng.random((per, s)) * e)
            loc = np.round((rng.random((per, s)) - 0.5) * 64) / 64
            # project loc onto the plane normal . loc = offset along the largest axis
            ax = int(np.argmax(np.abs(nrm)))
            rest = loc @ nrm - nrm[ax] * loc[:, ax]
            loc[:, ax] = (float(plane.offset) - rest) / nrm[ax]
            cand = site + loc
            ok = np.all(np.abs(cand - np.round(cand * 64) / 64) == 0, axis=1)
            pts.append(cand[ok])
    # 4) out-of-range (negative and beyond the extent)
    pts.append(_f32((rng.random((per, s)) - 0.5) * 4 * e))
    out = np.concatenate(pts, axis=0)
    return _f32(out)


def grid_points(space, extents, rng, count):
    e = np.array(extents, dtype=np.float64)
    return np.floor(rng.random((count, space.dim)) * e * 64) / 64


def falg(space, data, pts):
    n = space.stencil_size
    prog = generate(space, GenConfig(ScheduleParams(1, n, "branchy")))
    c = Counter()
    interpret_batch(prog, pts, data, counter=c)
    return sum(c[op] for op in FP_OPS) / len(pts)


def make_one(name, space, text, extents, out_dir, npts=2000, seed=0):
    rng = np.random.default_rng(1234 + seed)
    vol = make_volume(space, extents, seed=seed, float_width="f32")
    data64 = DataVolume([a.astype(np.float64) for a in vol.arrays])
    uni = _f32(sample_points(space, vol, npts, seed=seed + 1))
    sets = {
        "uniform": uni,
        "grid": _f32(grid_points(space, extents, rng, npts // 4)),
        "adversarial": adversarial_points(space, extents, rng, npts // 2),
    }
    arrays = {f"vol_{i}": a for i, a in enumerate(vol.arrays)}
    for key, xs in sets.items():
        arrays[f"{key}_xs"] = xs.astype(np.float32)
        arrays[f"{key}_value"] = ref_oracle.reference_eval_batch(space, xs, data64)
        ks, subs = [], []
        for off in space.lattice.cosets:
            xl = xs - np.array([float(q) for q in off])
            k, xloc = ref_oracle._rho(space, xl)
            ks.append(k.astype(np.int32))
            subs.append(ref_oracle._membership(space, xloc).astype(np.int32))
        arrays[f"{key}_k"] = np.stack(ks)
        arrays[f"{key}_sub"] = np.stack(subs)
    # generated-code execution (f64 and f32 programs) on the uniform set
    n = space.stencil_size
    for fw in ("f64", "f32"):
        prog = generate(space, GenConfig(ScheduleParams(1, n, "predicated"), float_width=fw))
        arrays[f"uniform_interp_{fw}"] = interpret_batch(prog, uni, data64).astype(np.float64)
    np.savez_compressed(out_dir / f"{name}.npz", **arrays)
    (out_dir / "spaces").mkdir(exist_ok=True)
    (out_dir / "spaces" / f"{name}.json").write_text(text)
    return falg(space, data64, uni[: min(4096, len(uni))])


def main(argv):
    out = HERE
    falgs = {}
    fpath = out / "falg.json"
    if fpath.exists():
        falgs = json.loads(fpath.read_text())
    jobs = []
    for name, ext in FIXTURES.items():
        space = parse_space(fixture_text(name))
        jobs.append((name, space, serialize_space(space), ext))
    for path in argv:
        text = Path(path).read_text()
        space = parse_space(text)  # the reference validates our producer's output
        meta = json.loads(text).get("x_golden", {})
        ext = tuple(meta.get("extents", [6] * space.dim))
        jobs.append((space.name, space, text, ext))
    for name, space, text, ext in jobs:
        npts = 2000 if space.stencil_size * space.ncosets <= 64 else 600
        falgs[name] = make_one(name, space, text, ext, out, npts=npts)
        print(f"{name}: F_alg = {falgs[name]:.2f} FP ops/query")
    fpath.write_text(json.dumps(falgs, indent=1, sort_keys=True) + "\n")
    return 0


if __name__ == "__main__":
    raise SystemExit(main(sys.argv[1:]))
