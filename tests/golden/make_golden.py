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
sys.path.insert(0, str(HERE.parents[1]))
from tests.adversarial import adversarial_points  # noqa: E402  (the generator, shared with the GPU tests)
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


def grid_points(space, extents, rng, count):
    e = np.array(extents, dtype=np.float64)
    return np.floor(rng.random((count, space.dim)) * e * 64) / 64


def falg(space, data, pts):
    n = space.stencil_size
    prog = generate(space, GenConfig(ScheduleParams(1, n, "branchy")))
    c = Counter()
    interpret_batch(prog, pts, data, counter=c)
    return sum(c[op] for op in FP_OPS) / len(pts)


# -- extension spaces (per-polynomial stencil sizes, > 32 planes) -------------------------
#
# The reference's evaluator handles these (oracle.py:77-104 fetches sub.stencil per
# region; sign vectors are int64), but its validator -- and so parse_space and generate --
# rejects them (model.py:365, :466-468).  Goldens come from `_parse_document` spaces and
# the reference oracle.  F_alg (the dynamic FP-op count of the reference's canonical
# branchy m=1 program) is measured on a SURROGATE the reference generator accepts: every
# sub-region's stencil is padded to the largest size with extra distinct sites whose
# symbols enter the polynomial as the single term 1 * c_j, and the generator's validator is
# told to ignore only the plane-count rule.  With m = 1 each padding symbol is its own chunk,
# i.e. a fixed number of extra FP ops per evaluated (query, coset) pair; that number is
# measured on a uniform space (pad_cost) and subtracted exactly.

EXTENSION_ERRORS = ("stencil sizes differ", "planes exceed the 32-bit")


def parse_extension_space(text):
    """(space, is_extension): parse_space, or _parse_document when the only invariant
    errors are the two extension rules."""
    import splinegen.model as smodel
    try:
        return parse_space(text), False
    except smodel.InvariantError as e:
        bad = [d for d in e.diagnostics if not any(k in d.message for k in EXTENSION_ERRORS)]
        if bad:
            raise
    doc = json.loads(text, parse_float=smodel._reject_float)
    return smodel._parse_document(doc), True


def _pad_space(space, n_to):
    """Uniform-stencil surrogate: stencils padded to n_to sites, psi_i += sum_pad 1 * c_j."""
    import dataclasses
    from fractions import Fraction
    from splinegen.poly import Poly
    from splinegen.model import RefPoly
    s = space.dim
    subs, ref_polys = [], list(space.ref_polys)
    done = set()
    for sub in space.subregions:
        have = len(sub.stencil)
        extra = tuple(tuple([1000 + j] + [0] * (s - 1)) for j in range(have, n_to))
        subs.append(dataclasses.replace(sub, stencil=tuple(sub.stencil) + extra))
        if sub.psi_index not in done:
            done.add(sub.psi_index)
            terms = dict(ref_polys[sub.psi_index].poly.terms)
            for j in range(have, n_to):
                terms[((0,) * s, j)] = Fraction(1)
            ref_polys[sub.psi_index] = RefPoly(Poly(s, terms))
    return dataclasses.replace(space, subregions=tuple(subs), ref_polys=tuple(ref_polys))


def _falg_relaxed(space, data, pts):
    """falg() with the generator's validator ignoring the plane-count rule only."""
    import splinegen.codegen as scodegen
    orig = scodegen.validate_space

    def relaxed(sp):
        return [d for d in orig(sp) if "planes exceed the 32-bit" not in d.message]
    scodegen.validate_space = relaxed
    try:
        return falg(space, data, pts)
    finally:
        scodegen.validate_space = orig


def pad_cost():
    """FP ops one padding symbol adds per evaluated (query, coset): measured on the
    reference's trilinear_voronoi fixture padded by 1 and by 3 sites."""
    space = parse_space(fixture_text("trilinear_voronoi"))
    vol = make_volume(space, (6, 6, 6), seed=0, float_width="f32")
    data = DataVolume([a.astype(np.float64) for a in vol.arrays])
    pts = _f32(sample_points(space, vol, 512, seed=1))
    n = space.stencil_size
    f0 = falg(space, data, pts)
    f1 = falg(_pad_space(space, n + 1), data, pts)
    f3 = falg(_pad_space(space, n + 3), data, pts)
    per = (f1 - f0) / space.ncosets
    assert abs((f3 - f0) / space.ncosets - 3 * per) < 1e-9, (f0, f1, f3)
    return per


def falg_extension(space, data, pts):
    """F_alg of a per-polynomial-stencil space (see above)."""
    n = max(len(sb.stencil) for sb in space.subregions)
    fpad = _falg_relaxed(_pad_space(space, n), data, pts)
    # padding symbols per query: sum over cosets of (n - n_psi(sub(query, coset)))
    miss = 0
    for off in space.lattice.cosets:
        xl = pts - np.array([float(q) for q in off])
        _, xloc = ref_oracle._rho(space, xl)
        sub = ref_oracle._membership(space, xloc)
        sizes = np.array([len(sb.stencil) for sb in space.subregions])
        miss += float((n - sizes[sub]).sum())
    return fpad - pad_cost() * miss / len(pts)


def make_one(name, space, text, extents, out_dir, npts=2000, seed=0, extension=False):
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
    # generated-code execution (f64 and f32 programs) on the uniform set -- not for
    # extension spaces, which the reference generator refuses
    n = max(len(sb.stencil) for sb in space.subregions)
    if not extension:
        for fw in ("f64", "f32"):
            prog = generate(space, GenConfig(ScheduleParams(1, n, "predicated"), float_width=fw))
            arrays[f"uniform_interp_{fw}"] = interpret_batch(prog, uni, data64).astype(np.float64)
    np.savez_compressed(out_dir / f"{name}.npz", **arrays)
    (out_dir / "spaces").mkdir(exist_ok=True)
    (out_dir / "spaces" / f"{name}.json").write_text(text)
    fpts = uni[: min(4096, len(uni))]
    return falg_extension(space, data64, fpts) if extension else falg(space, data64, fpts)


def main(argv):
    out = HERE
    falgs = {}
    fpath = out / "falg.json"
    if fpath.exists():
        falgs = json.loads(fpath.read_text())
    jobs = []
    only = os.environ.get("GOLDEN_ONLY_EXTRA") == "1"
    for name, ext in ({} if only else FIXTURES).items():
        space = parse_space(fixture_text(name))
        jobs.append((name, space, serialize_space(space), ext, False))
    for path in argv:
        text = Path(path).read_text()
        # the reference validates our producer's output (extension spaces: every rule
        # but the two extension ones, see parse_extension_space)
        space, ext_space = parse_extension_space(text)
        meta = json.loads(text).get("x_golden", {})
        ext = tuple(meta.get("extents", [6] * space.dim))
        jobs.append((space.name, space, text, ext, ext_space))
    for name, space, text, ext, ext_space in jobs:
        nmax = max(len(sb.stencil) for sb in space.subregions)
        npts = 2000 if nmax * space.ncosets <= 64 else 600
        falgs[name] = make_one(name, space, text, ext, out, npts=npts, extension=ext_space)
        print(f"{name}: F_alg = {falgs[name]:.2f} FP ops/query")
    fpath.write_text(json.dumps(falgs, indent=1, sort_keys=True) + "\n")
    return 0




# -- gradient work (bench configs that also return grad f) ---------------------------------


def _tree_ops(node):
    """fadd + fmul nodes of a reference Horner tree (what _tree_value emits, codegen.py:318-328)."""
    from splinegen.poly import Add, Mul
    if isinstance(node, (Add, Mul)):
        return 1 + _tree_ops(node.left) + _tree_ops(node.right)
    return 0


def falg_gradient_extra(space, pts):
    """FP ops per query the gradient adds to F_alg, by the reference's own counting rule:
    for every (query, coset) the m=1 chunked greedy-Horner programs of the three partial
    derivatives d psi / d u_k of the selected reference polynomial (the reference's
    Poly.differentiate + group_polynomial + horner_factorize, poly.py:169-376; one fadd per
    chunk accumulation as in _run_plan, codegen.py:332-356) plus grad_x = T^T grad_u
    (3 x (3 fmul + 2 fadd) per coset).  The reference itself has no gradient program."""
    from splinegen.poly import group_polynomial, horner_factorize
    ops = []
    for rp, sub0 in zip(space.ref_polys, [next(sb for sb in space.subregions if sb.psi_index == i)
                                          for i in range(len(space.ref_polys))]):
        total = 0
        n = len(sub0.stencil)
        for k in range(space.dim):
            dp = rp.poly.differentiate(k)
            cs = group_polynomial(dp, 1, range(n))
            used = 0
            for poly, _blk in cs.chunks:
                if poly.terms:
                    total += _tree_ops(horner_factorize(poly))
                    used += 1
            total += max(0, used - 1)
        ops.append(total + space.dim * (2 * space.dim - 1))
    acc = 0.0
    for off in space.lattice.cosets:
        xl = pts - np.array([float(q) for q in off])
        _, xloc = ref_oracle._rho(space, xl)
        sub = ref_oracle._membership(space, xloc)
        psi = np.array([sb.psi_index for sb in space.subregions])[sub]
        acc += float(np.array(ops)[psi].sum())
    return acc / len(pts)


def grad_main(names):
    """falg.json["<space>+grad"] = F_alg + falg_gradient_extra, for the gradient configs."""
    fpath = HERE / "falg.json"
    falgs = json.loads(fpath.read_text())
    for name in names:
        text = (HERE / "spaces" / f"{name}.json").read_text()
        space, _ = parse_extension_space(text)
        z = np.load(HERE / f"{name}.npz")
        pts = z["uniform_xs"].astype(np.float64)
        falgs[f"{name}+grad"] = round(falgs[name] + falg_gradient_extra(space, pts), 3)
        print(f"{name}+grad: {falgs[name + '+grad']:.2f} FP ops/query")
    fpath.write_text(json.dumps(falgs, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    if sys.argv[1:2] == ["--grad"]:
        raise SystemExit(grad_main(sys.argv[2:]))
    raise SystemExit(main(sys.argv[1:]))
