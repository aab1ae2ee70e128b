"""Hardware linear-fetch variant.

The paper's CUDA backend can replace pairs of neighbouring coefficient reads by one
texture fetch with hardware linear filtering: for two sites a, a+1 on one axis with
weights w_a, w_{a+1} of equal sign,

    w_a c_a + w_{a+1} c_{a+1} = g * lerp(c_a, c_{a+1}, h),  g = w_a + w_{a+1},  h = w_{a+1} / g,

and the texture unit evaluates the lerp.  For a tensor-product spline every stencil
weight factors per axis, W_p(u) = prod_a w_{a,p_a}(u_a), so the pairing applies on every
axis at once: the tricubic's 64 point reads become 8 trilinear fetches ("we reduce 64
fetches to 8 via the linear fetch trick").  "Parts of the polynomial are
computed prior to the fetches": the 1-D weights are Horner polynomials in u.

This module derives the per-axis weight polynomials from the space itself (exact rational
rank-1 factorisation of every site's weight polynomial; `separable_plan` refuses spaces
whose weights do not factor -- box and Voronoi splines on BCC/FCC) and emits an sm_100a
kernel that fetches through texture objects (3-D cudaArrays, wrap addressing = the
reference's periodic `fetch`, `src/ir.py:555-558`; the C ABI builds them from the volume).

Accuracy: the texture unit quantises the lerp fraction to 8 bits (1/256), so every fetch
is off by up to |c_{a+1} - c_a| / 512 per filtered axis.  The variant therefore CANNOT
meet the north star's 1e-5 (the reference marks it out of scope); it is opt-in
(`GenConfig(fetch="linear")`) and its parity test states its own bound
(tests/test_linfetch.py).  Selection (k, sub-region) stays bit-exact: floor / round-half-away
in fp64 like the oracle (`src/oracle.py:34-53`).
"""

from __future__ import annotations

import itertools
from fractions import Fraction

from . import exact
from .model import PARALLELEPIPED, SplineSpace
from .poly import NO_SYMBOL

ENTRY = "sg_eval_kernel"


class LinearFetchPlan:
    """Per axis a: the 1-D stencil offsets v_lo..v_hi and the weight polynomial of each
    offset (ascending Fraction coefficients), with W_p(u) = prod_a w[a][p_a](u_a) exactly;
    `pairs[a]` lists (v, paired) -- `paired` True when v and v+1 share one filtered fetch."""

    def __init__(self, dim, vlo, weights, pairs):
        self.dim = dim
        self.vlo = vlo            # per axis: smallest stencil offset
        self.weights = weights    # per axis: [coeffs of w_{vlo}, coeffs of w_{vlo+1}, ...]
        self.pairs = pairs        # per axis: [(v, paired), ...]

    @property
    def fetches(self):
        n = 1
        for p in self.pairs:
            n *= len(p)
        return n

    @property
    def point_reads(self):
        n = 1
        for w in self.weights:
            n *= len(w)
        return n


def _rank1(tensor, dim):
    """Exact factorisation T[e] = prod_a f_a[e_a] of a coefficient tensor {exps: q} (or
    None).  Factors 1..dim-1 are normalised to leading (lowest-degree nonzero) coefficient
    1; factor 0 carries the scale -- so the factorisation is unique."""
    if not tensor:
        return None
    pivot = min(tensor)
    pv = tensor[pivot]
    degs = [max(e[a] for e in tensor) for a in range(dim)]
    factors = []
    for a in range(dim):
        f = []
        for k in range(degs[a] + 1):
            e = list(pivot)
            e[a] = k
            f.append(tensor.get(tuple(e), Fraction(0)))
        factors.append(f)
    for a in range(1, dim):
        factors[a] = [c / pv for c in factors[a]]
    for a in range(1, dim):
        lead = next(c for c in factors[a] if c != 0)
        factors[a] = [c / lead for c in factors[a]]
        factors[0] = [c * lead for c in factors[0]]
    if _outer(factors, dim) != tensor:
        return None
    return [_trim(f) for f in factors]


def _trim(c):
    c = list(c)
    while len(c) > 1 and c[-1] == 0:
        c.pop()
    return c


def _peval(c, u):
    acc = Fraction(0)
    for q in reversed(c):
        acc = acc * u + q
    return acc


def _outer(factors, s):
    out = {(): Fraction(1)}
    for a in range(s):
        nxt = {}
        for e, q in out.items():
            for k, c in enumerate(factors[a]):
                if c != 0:
                    nxt[e + (k,)] = q * c
        out = nxt
    return {e: q for e, q in out.items() if q != 0}


def _ratio(f, g):
    """The scalar lam with f = lam * g exactly (or None)."""
    f, g = _trim(f), _trim(g)
    if len(f) != len(g):
        return None
    k = next((i for i, c in enumerate(g) if c != 0), None)
    if k is None:
        return None
    lam = f[k] / g[k]
    return lam if all(a == lam * b for a, b in zip(f, g)) else None


def separable_plan(space: SplineSpace) -> LinearFetchPlan:
    """The per-axis factorisation of a tensor-product space (ValueError otherwise)."""
    s = space.dim
    if s > 3:
        raise ValueError("linear fetch: textures are 1-, 2- or 3-D")
    rm = space.region_map
    if rm.shape == PARALLELEPIPED and not exact.is_identity(rm.basis):
        raise ValueError("linear fetch needs an identity region-of-evaluation basis")
    if len(space.ref_polys) != 1 or len(space.subregions) != 1:
        raise ValueError("linear fetch needs one sub-region and one reference polynomial "
                         "(a tensor-product spline)")
    sub = space.subregions[0]
    if not exact.is_identity(sub.transform) or any(Fraction(v) != 0 for v in sub.shift):
        raise ValueError("linear fetch needs an identity sub-region transform")
    sten = [tuple(int(v) for v in site) for site in sub.stencil]
    per_site = [dict() for _ in sten]
    for (exps, ci), q in space.ref_polys[0].poly.terms.items():
        if ci == NO_SYMBOL:
            raise ValueError("linear fetch: the polynomial has a data-free term")
        per_site[ci][tuple(exps)] = Fraction(q)
    vlo = [min(p[a] for p in sten) for a in range(s)]
    vhi = [max(p[a] for p in sten) for a in range(s)]
    full = 1
    for a in range(s):
        full *= vhi[a] - vlo[a] + 1
    if len(set(sten)) != len(sten) or full != len(sten):
        raise ValueError("linear fetch needs a full rectangular stencil")
    index = {p: j for j, p in enumerate(sten)}
    facs = {}
    for j, p in enumerate(sten):
        f = _rank1({e: q for e, q in per_site[j].items() if q != 0}, s)
        if f is None:
            raise ValueError(f"linear fetch: the weight of site {p} does not factor per axis "
                             "(not a tensor-product spline)")
        facs[p] = f
    r = tuple(vlo)   # corner site

    def line(a, v):
        p = list(r)
        p[a] = v
        return tuple(p)
    # axis 0 carries the scale of the corner line; axes >= 1 keep their normalised factors,
    # scaled by how the axis-0 factor changes along their line through the corner
    weights = [[facs[line(0, v)][0] for v in range(vlo[0], vhi[0] + 1)]]
    for a in range(1, s):
        col = []
        for v in range(vlo[a], vhi[a] + 1):
            lam = _ratio(facs[line(a, v)][0], facs[r][0])
            if lam is None:
                raise ValueError("linear fetch: the axis factors are not separable")
            col.append([lam * c for c in facs[line(a, v)][a]])
        weights.append(col)
    for p, j in index.items():
        if _outer([weights[a][p[a] - vlo[a]] for a in range(s)], s) != \
                {e: q for e, q in per_site[j].items() if q != 0}:
            raise ValueError(f"linear fetch: site {p} is not the product of the axis factors")
    # local coordinate range of the cell: [0, 1) after floor, [-1/2, 1/2] after rounding
    u0 = Fraction(0) if rm.rounding == "floor" else Fraction(-1, 2)
    pairs = []
    for a in range(s):
        nv = vhi[a] - vlo[a] + 1
        lst = []
        v = 0
        while v < nv:
            ok = v + 1 < nv and _same_sign(weights[a][v], weights[a][v + 1], u0)
            lst.append((vlo[a] + v, ok))
            v += 2 if ok else 1
        pairs.append(lst)
    return LinearFetchPlan(s, vlo, weights, pairs)


def _same_sign(f, g, u0, samples=64):
    """Weights of equal sign on the local cell [u0, u0 + 1] (sampled at 65 points)."""
    for k in range(samples + 1):
        u = u0 + Fraction(k, samples)
        if _peval(f, u) * _peval(g, u) < 0:
            return False
    return True


def _horner(coeffs, var, fw="f32"):
    from .cudagen import flit
    cs = [flit(c, fw) for c in coeffs]
    expr = cs[-1]
    for c in reversed(cs[:-1]):
        expr = f"fmaf({expr}, {var}, {c})"
    return expr


def generate_linear(space, cfg, ext):
    """The linear-fetch kernel for `space` (per-coset extents `ext`) as a CudaProgram
    (mode "linear": the C ABI binds one 2-D/3-D texture per coset, sg_eval passes them)."""
    from dataclasses import replace

    from .cudagen import ENTRY as CENTRY
    from .cudagen import F32, CudaProgram, dlit
    from .model import ROUND_NEAREST
    assert CENTRY == ENTRY
    if cfg.float_width != F32:
        raise ValueError("linear fetch filters f32 textures (float_width='f32')")
    if cfg.grad:
        raise ValueError("linear fetch: derivative weights change sign inside a pair, so the "
                         "gradient cannot be filtered (grad=False)")
    if cfg.mode != "direct" or cfg.pack != 1:
        raise ValueError("linear fetch is a direct-mode variant")
    plan = separable_plan(space)
    s, M = space.dim, space.ncosets
    if any(len(e) != s for e in ext) or len(ext) != M:
        raise ValueError(f"extents must give {s} values for each of {M} cosets")
    rm = space.region_map
    rounding = rm.rounding if rm.shape == PARALLELEPIPED else ROUND_NEAREST
    B = cfg.block
    ldf = "__ldcs" if cfg.stream == "cs" else "__ldg"
    L = []
    A = L.append
    A(f"// generated by paper_2102_08518_b200.linfetch for space '{space.name}'")
    A(f"// hardware linear fetch: {plan.point_reads} point reads -> {plan.fetches} filtered "
      f"texture fetches per coset; block={B} dbg={int(cfg.dbg)}")
    A(f"// extents={tuple(ext)} rounding={rounding}")
    A("struct SgTex { unsigned long long t[8]; };")
    A(f"extern \"C\" __global__ void __launch_bounds__({B}) {ENTRY}(")
    A("    const float* __restrict__ xs, long long n, float* __restrict__ out, float* __restrict__ grad,")
    A("    int* __restrict__ dbg, unsigned* __restrict__ err, SgTex tex) {")
    A(f"  for (long long qi = (long long)blockIdx.x * {B} + threadIdx.x; qi < n;")
    A(f"       qi += (long long)gridDim.x * {B}) {{")
    for d in range(s):
        A(f"    const double x{d} = (double){ldf}(&xs[qi * {s} + {d}]);")
    A("    float acc = 0.0f;")
    cos = [tuple(Fraction(v) for v in c) for c in space.lattice.cosets]
    for l in range(M):
        A(f"    {{  // coset {l}")
        for d in range(s):
            o = cos[l][d]
            A(f"      const double xl{d} = " + (f"x{d};" if o == 0 else f"__dsub_rn(x{d}, {dlit(o)});"))
            if rounding == ROUND_NEAREST:
                A(f"      const long long k{d} = __double2ll_rz(__dadd_rn(xl{d}, copysign(0.5, xl{d})));")
            else:
                A(f"      const long long k{d} = __double2ll_rd(xl{d});")
            A(f"      const float u{d} = (float)__dsub_rn(xl{d}, (double)k{d});")
            E = ext[l][d]
            A(f"      long long kr{d} = k{d} % {E}LL; if (kr{d} < 0) kr{d} += {E}LL;")
            A(f"      const float kf{d} = (float)kr{d};")
        if cfg.dbg:
            for d in range(s):
                A(f"      dbg[(qi * {M} + {l}) * {s + 1} + {d}] = (int)k{d};")
            A(f"      dbg[(qi * {M} + {l}) * {s + 1} + {s}] = 0;")
        # per axis: 1-D weights (Horner in u), then per pair (g, texel coordinate)
        for d in range(s):
            for vi, w in enumerate(plan.weights[d]):
                A(f"      const float w{d}_{vi} = {_horner(w, f'u{d}')};")
            for pi, (v, paired) in enumerate(plan.pairs[d]):
                vi = v - plan.vlo[d]
                E = ext[l][d]
                if paired:
                    A(f"      const float g{d}_{pi} = w{d}_{vi} + w{d}_{vi + 1};")
                    A(f"      const float h{d}_{pi} = g{d}_{pi} != 0.0f ? __fdiv_rn(w{d}_{vi + 1}, g{d}_{pi}) : 0.0f;")
                    A(f"      const float c{d}_{pi} = (kf{d} + ({float(v) + 0.5!r}f + h{d}_{pi})) * (1.0f / {E}.0f);")
                else:
                    A(f"      const float g{d}_{pi} = w{d}_{vi};")
                    A(f"      const float c{d}_{pi} = (kf{d} + {float(v) + 0.5!r}f) * (1.0f / {E}.0f);")
        A(f"      const unsigned long long tx = tex.t[{l}];")
        for combo in itertools.product(*[range(len(plan.pairs[d])) for d in range(s)]):
            wexpr = " * ".join(f"g{d}_{combo[d]}" for d in range(s))
            coords = [f"c{d}_{combo[d]}" for d in range(s)]
            if s == 1:
                fetch = f"tex1D<float>(tx, {coords[0]})"
            elif s == 2:
                fetch = f"tex2D<float>(tx, {coords[1]}, {coords[0]})"
            else:
                fetch = f"tex3D<float>(tx, {coords[2]}, {coords[1]}, {coords[0]})"
            A(f"      acc = fmaf({wexpr}, {fetch}, acc);")
        A("    }")
    A("    __stcs(&out[qi], acc);" if cfg.stream == "cs" else "    out[qi] = acc;")
    A("  }")
    A("}")
    src = "\n".join(L) + "\n"
    ext_t = tuple(tuple(int(v) for v in e) for e in ext)
    return CudaProgram(
        name=space.name, source=src, entry=ENTRY, dim=s, ncosets=M, float_width=F32,
        block=B, halo=0, extents=ext_t, padded_extents=ext_t, has_grad=False,
        has_dbg=cfg.dbg, config=replace(cfg), space=space, mode="linear",
        rounding=(0 if rounding == "floor" else 1),
        meta={"fetch_mode": "linear", "K": 1, "nsub": 1, "fetches": plan.fetches,
              "point_reads": plan.point_reads, "reach": 0})
