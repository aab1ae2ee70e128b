"""CUDA C++ emission: spline space + variant knobs -> one sm_100a kernel.

This replaces the reference's lowering + LLVM emission
(pkg/src/splinegen/codegen.py:85-510 -> emit.py:43-262).  The generated kernel
evaluates Algorithm 1 for ONE query per thread:

  per coset l (unrolled, or a rolled loop -- codegen.py:406-469):
    xl  = x - offset_l                                 (fp64)
    k   = rnd(B^-1 xl) mapped back by B; x_loc = xl - k  (fp64, codegen.py:190-226)
    q   = sum_i [normal_i . x_loc >= offset_i] << i      (fp64, codegen.py:230-250)
    sub = sigma[q mod p]; sigma == -1 sets the error word
    u   = T_sub x_loc + t'_sub                          (codegen.py:281-304)
    c_j = V_l[wrap(k) + pi_sub[j]]  (ghost halo: one wrap per coset, not per fetch)
    g   = psi_{psi(sub)}(u, c)  via the scheduled chunk trees  (codegen.py:332-402)
  f = sum_l g_l

Selection (rho, plane tests) runs in fp64 op-for-op like the fp64 oracle
(oracle.py:34-74), which makes k and the sub-region bit-exact against it
(SURVEY H2); polynomial evaluation runs in the program dtype (f32 or f64).

Variant knobs (GenConfig): the reference's (m, d, branch_mode, refetch_tables,
float_width, unroll_cosets) plus GPU ones -- `form` ("horner": the reference's
greedy Horner trees per chunk; "sites": per-site weight polynomials
w_j(u) = d psi / d c_j in Horner form, then sum c_j w_j), `coeffs` ("imm":
hard-coded FMA immediates; "lut": coefficients in a __constant__ lookup table
read as constant-bank operands), `block`, `grad`, `dbg`.
"""

from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass, field, replace
from fractions import Fraction

import numpy as np

from . import exact
from .model import PARALLELEPIPED, ROUND_NEAREST, SplineSpace, validate_space
from .poly import NO_SYMBOL, Add, Const, Mul, Poly, Sym, Var, group_polynomial, horner_factorize
from .schedule import BRANCHY, COMPUTE, FETCH, PREDICATED, ScheduleParams, schedule_pipeline

F64 = "f64"
F32 = "f32"
ENTRY = "sg_eval_kernel"
FORMS = ("horner", "sites", "sym")
COEFFS = ("imm", "lut", "table")


@dataclass(frozen=True)
class GenConfig:
    """Reference fields (codegen.py:38-46) + B200 kernel-variant knobs."""
    params: ScheduleParams
    # None -> the reference's default (f64, codegen.py:38-46) for direct-mode kernels; the
    # f32-only execution modes (binned / sorted / render, pack=2) default to f32
    float_width: str | None = None
    unroll_cosets: bool = True
    form: str = "horner"
    coeffs: str = "imm"
    block: int = 128
    grad: bool = False
    dbg: bool = False
    min_blocks: int = 0          # __launch_bounds__ second argument (0 = let ptxas pick)
    mode: str = "direct"         # "direct": gathers through L1/L2; "binned": bin + smem bricks
    bin: int = 0                 # binned: bin edge in lattice cells (multiple of 4; 0 = auto)
    chunk: int = 4096            # binned: queries per CTA work item (a bin is split in chunks)
    brick_budget: int = 112 * 1024   # binned auto-bin: shared-memory budget for the bricks
    stage: str = "tma"           # binned: brick staging, "tma" (cp.async.bulk.tensor) | "ldg"
    tile: int = 0                # sorted: queries per CTA tile (0 = auto: 2 CTAs / SM of smem)
    stream: str = "cs"           # query/result cache policy: "cs" (evict-first) | "default"
    select: str = "auto"         # selection arithmetic: "f64" | "int" (2^-30 fixed point) | "auto"
    sigma_smem: int = 4096       # sigma tables up to this many entries are staged in smem
    pack: int = 1                # 2: two queries per thread, polynomial FP in packed f32x2 (FFMA2)
    prefetch: int = 0            # sorted: load the next pair's record + coefficients one iteration ahead
    radix: int = 0               # 1: sub-region via a mixed-radix index of the plane-family counts
    rank: str = "match"          # sorted: rank in the psi class by "match" (warp-aggregated) | "atomic"
    presort: int = 0             # sorted: bin edge (cells) of a locality pre-sort of the queries (0 = off)
    tpairs: int = 1              # sorted + table + tloop: 2 = two pairs of one polynomial per thread
    tchunk: int = 0              # table + tloop: monomials per pass (0 = all up to 96, else 80)
    cmajor: int = 0              # sorted: evaluate class by class (1; 2 = with a CTA barrier between
                                 # classes) so the warps of an SM execute one polynomial's code
    qhoist: int = 0              # sorted: issue all of a thread's tile query loads before the
                                 # first selection (one memory latency per tile, not per query)
    tloop: int = 0               # coeffs="table": 1 = a runtime loop over the stencil sites (code
                                 # shared by every reference polynomial: no instruction-cache
                                 # pressure for large polynomials), 0 = fully unrolled
    fetch_offsets: str = "affine"  # sorted mode, per-polynomial stencils: "affine" (offsets from
                                   # the arm's reference stencil + 4 ints per sub-region) | "table"
    cflip: int = 0               # sorted + cmajor=3: alternate the psi order tile by tile (the
                                 # last polynomial's code is still hot when the next tile starts)
    gtables: str = ""            # sorted / direct / render: comma-separated shared tables read
                                 # from global memory (L1-cached __ldg) instead of being staged in
                                 # shared memory, e.g. "sg_Tq" -- frees shared memory so the L1
                                 # carve-out stays larger at a given tile size
    fetch: str = "point"         # "linear": hardware-filtered texture fetches for tensor-product
                                 # spaces (opt-in, ~1e-3 accurate: linfetch.py)

    def __post_init__(self):
        if self.float_width is None:
            object.__setattr__(self, "float_width",
                               F64 if (self.mode == "direct" and self.pack == 1
                                       and self.fetch == "point") else F32)
        if self.fetch not in ("point", "linear"):
            raise ValueError("fetch must be 'point' or 'linear'")
        if self.fetch_offsets not in ("affine", "table"):
            raise ValueError("fetch_offsets must be 'affine' or 'table'")
        if self.float_width not in (F64, F32):
            raise ValueError(f"float width must be f64 or f32, not {self.float_width!r}")
        if self.form not in FORMS:
            raise ValueError(f"form must be one of {FORMS}")
        if self.coeffs not in COEFFS:
            raise ValueError(f"coeffs must be one of {COEFFS}")
        if self.block % 32 or not 32 <= self.block <= 1024:
            raise ValueError("block must be a multiple of 32 in [32, 1024]")
        if self.mode not in ("direct", "binned", "sorted", "render"):
            raise ValueError("mode must be 'direct', 'binned', 'sorted' or 'render'")
        if self.pack not in (1, 2):
            raise ValueError("pack must be 1 or 2")
        if self.stream not in ("cs", "default"):
            raise ValueError("stream must be 'cs' or 'default'")
        if self.select not in ("auto", "f64", "int"):
            raise ValueError("select must be 'auto', 'f64' or 'int'")
        if self.mode in ("sorted", "render") and (self.tile % self.block or self.tile > 8192 or self.tile < 0):
            raise ValueError("sorted mode: tile must be a multiple of block and <= 8192")
        if self.stage not in ("tma", "ldg", "l1"):
            raise ValueError("stage must be 'tma', 'ldg' or 'l1' (no staging: sorted queries, L1 gathers)")


def default_config(space: SplineSpace, **kw) -> GenConfig:
    """The paper's GPU default: m = 1, d = n, predicated."""
    n = space.stencil_size
    params = kw.pop("params", None) or ScheduleParams(1, n, PREDICATED)
    return GenConfig(params=params, **kw)


# -- literals ------------------------------------------------------------------


def flit(q, fw: str) -> str:
    """Exact hex literal of the rational rounded to the program float type."""
    v = float(Fraction(q))
    if fw == F32:
        v32 = float(np.float32(v))
        if v32 == 0.0:
            return "0.0f"
        return f"{v32.hex()}f"
    if v == 0.0:
        return "0.0"
    return v.hex()


def dlit(q) -> str:
    v = float(Fraction(q))
    return "0.0" if v == 0.0 else v.hex()


# -- derived tables --------------------------------------------------------------


@dataclass
class Tables:
    s: int
    M: int
    nsub: int
    n: int
    K: int
    cosets: list            # M x s Fractions
    planes: list            # (normal Fractions, offset Fraction)
    modulus: int
    sigma: list
    compress: bool
    transforms: list        # nsub x (s x s Fractions)
    tshift: list            # nsub x s Fractions  (t' = -T t)
    stencils: list          # nsub x n x s ints
    psi: list               # nsub ints
    halo: int
    uniform_T: bool
    uniform_tp: bool
    uniform_stencil: bool
    uniform_psi: bool
    affine: list | None     # per sub: (A int s x s, b int s) with pi_sub[j] = A ref[j] + b
    ref_stencil: list       # n x s
    n_psi: list = None      # K: stencil size of each reference polynomial (n = the largest)
    # per reference polynomial its stencil (that of its first sub-region) and per sub-region
    # (A, b) with pi_sub[j] = A ref_psi[psi_sub][j] + b (None when some sub has no such map)
    ref_psi: list = None
    paffine: list | None = None

    @property
    def uniform_n(self):
        return len(set(self.n_psi)) == 1


def _solve_affine(ref, sten, s):
    """Find integer A, b with sten[j] = A ref[j] + b for all j (or None)."""
    n = len(ref)
    if n == 0:
        return None
    # pick s independent difference vectors of ref
    diffs = [(j, tuple(ref[j][d] - ref[0][d] for d in range(s))) for j in range(1, n)]
    basis = []
    for j, v in diffs:
        cand = basis + [(j, v)]
        m = [list(map(Fraction, w)) for _, w in cand]
        # rank check via determinant of the Gram-like selection
        if _rank(m) == len(cand):
            basis = cand
        if len(basis) == s:
            break
    if len(basis) < s:
        # degenerate stencil (e.g. n <= s, or coplanar sites): A is not determined by the
        # sites, so the signed permutations (the producer's symmetry maps) are tried
        import itertools as _it
        for perm in _it.permutations(range(s)):
            for signs in _it.product((1, -1), repeat=s):
                A = [[signs[i] if perm[i] == j else 0 for j in range(s)] for i in range(s)]
                b = [sten[0][d] - sum(A[d][e] * ref[0][e] for e in range(s)) for d in range(s)]
                if all(tuple(sum(A[d][e] * ref[j][e] for e in range(s)) + b[d] for d in range(s))
                       == tuple(sten[j]) for j in range(n)):
                    return A, b
        return None
    R = [[Fraction(v[d]) for (_, v) in basis] for d in range(s)]   # columns = ref diffs
    S = [[Fraction(sten[j][d] - sten[0][d]) for (j, _) in basis] for d in range(s)]
    try:
        Rinv = exact.inverse(tuple(tuple(r) for r in R))
    except ValueError:
        return None
    A = exact.matmul(tuple(tuple(r) for r in S), Rinv)
    if not exact.is_int_mat(A):
        return None
    b = exact.sub(tuple(Fraction(v) for v in sten[0]), exact.matvec(A, ref[0]))
    if not exact.is_int_vec(b):
        return None
    for j in range(n):
        got = exact.add(exact.matvec(A, ref[j]), b)
        if tuple(int(v) for v in got) != tuple(sten[j]):
            return None
    return [[int(v) for v in row] for row in A], [int(v) for v in b]


def _rank(rows):
    a = [list(r) for r in rows]
    rank = 0
    ncol = len(a[0]) if a else 0
    for c in range(ncol):
        p = next((r for r in range(rank, len(a)) if a[r][c] != 0), None)
        if p is None:
            continue
        a[rank], a[p] = a[p], a[rank]
        for r in range(len(a)):
            if r != rank and a[r][c] != 0:
                f = a[r][c] / a[rank][c]
                a[r] = [x - f * y for x, y in zip(a[r], a[rank])]
        rank += 1
    return rank


def derive_tables(space: SplineSpace) -> Tables:
    s = space.dim
    subs = space.subregions
    transforms = [tuple(tuple(Fraction(v) for v in row) for row in sb.transform) for sb in subs]
    tshift = [exact.neg(exact.matvec(sb.transform, sb.shift)) for sb in subs]
    stencils = [[tuple(int(v) for v in site) for site in sb.stencil] for sb in subs]
    psi = [sb.psi_index for sb in subs]
    halo = max([abs(v) for st in stencils for site in st for v in site] + [0])
    ref = stencils[0]
    aff = []
    for st in stencils:
        r = _solve_affine(ref, st, s) if len(st) == len(ref) else None
        if r is None:
            aff = None
            break
        aff.append(r)
    # per reference polynomial: its stencil size (higher-order Voronoi splines carry
    # per-polynomial stencils; every sub-region of one polynomial has the same size)
    n_psi = [0] * len(space.ref_polys)
    for sb in subs:
        n_psi[sb.psi_index] = len(sb.stencil)
    ref_psi = [None] * len(space.ref_polys)
    for st, p_ in zip(stencils, psi):
        if ref_psi[p_] is None:
            ref_psi[p_] = st
    paff = []
    for st, p_ in zip(stencils, psi):
        r = _solve_affine(ref_psi[p_], st, s) if len(st) == len(ref_psi[p_]) else None
        if r is None:
            paff = None
            break
        paff.append(r)
    P = space.indexer.modulus
    Q = len(space.planes)
    return Tables(
        s=s, M=space.ncosets, nsub=len(subs), n=space.stencil_size, K=len(space.ref_polys),
        cosets=[tuple(Fraction(v) for v in c) for c in space.lattice.cosets],
        planes=[(tuple(Fraction(v) for v in p.normal), Fraction(p.offset)) for p in space.planes],
        modulus=P, sigma=list(space.indexer.sigma), compress=(Q > 0 and 2 ** Q > P),
        transforms=transforms, tshift=tshift, stencils=stencils, psi=psi, halo=halo,
        uniform_T=len(set(transforms)) == 1, uniform_tp=len(set(tshift)) == 1,
        uniform_stencil=len({tuple(x) for x in stencils}) == 1, uniform_psi=len(set(psi)) == 1,
        affine=aff, ref_stencil=ref, n_psi=n_psi, ref_psi=ref_psi, paffine=paff)


def plane_families(t: Tables) -> dict:
    """Families of parallel planes with offsets m_1..m_r * 2^-p (consecutive integers m,
    contiguous increasing bits): their r bits are one threshold count,
    cnt = clamp(floor(dot * 2^p) - m_1 + 1, 0, r) -- exact, because dot * 2^p is exact
    and comparing with integers commutes with floor.  normal -> (bit0, r, 2^p, m_1)."""
    fams = {}
    for i, (nrm, off) in enumerate(t.planes):
        fams.setdefault(nrm, []).append((i, off))
    counted = {}
    for nrm, lst in fams.items():
        if len(lst) < 3:
            continue
        idxs = [i for i, _ in lst]
        offs = [o for _, o in lst]
        if idxs != list(range(idxs[0], idxs[0] + len(idxs))):
            continue
        step = offs[1] - offs[0]
        if step <= 0 or any(offs[k + 1] - offs[k] != step for k in range(len(offs) - 1)):
            continue
        inv = 1 / step
        if inv.denominator != 1 or int(inv) & (int(inv) - 1):
            continue   # spacing must be 2^-p so the scaling is exact
        m1 = offs[0] * inv
        if m1.denominator != 1:
            continue
        counted[nrm] = (idxs[0], len(idxs), int(inv), int(m1))
    return counted


FIX = 30          # fixed-point fraction bits of the integer selection path
FIX_MIN = 2.0 ** -7   # |x| >= 2^-7: an fp32 x is a multiple of 2^-30 (ulp(2^-7) = 2^-30)


def int_selection_ok(space, t: Tables, fw: str) -> bool:
    """Can rho + plane tests run exactly in 2^-30 fixed point (int32)?

    For f32 queries x >= 2^-7 every quantity the fp64 oracle forms (x - l, the rounding,
    x_loc, small-integer plane dots, dot * 2^p) is a multiple of 2^-30 that fp64 holds
    exactly, so exact integer arithmetic on x * 2^30 reproduces it bit for bit
    (oracle.py:34-74).  Needs: identity region basis, coset offsets m * 2^-30 in
    [0, 1/2] (round) or [0, 1) (floor), integer plane normals and offsets m * 2^-30 with
    every |dot| < 2^31, family spacings 2^-p with p <= 30."""
    if fw != F32 or t.s > 3:
        return False
    rm = space.region_map
    if rm.shape == PARALLELEPIPED:
        if not exact.is_identity(rm.basis):
            return False
        rounding = rm.rounding
    else:
        rounding = ROUND_NEAREST
    hi = Fraction(1, 2) if rounding == ROUND_NEAREST else Fraction(1)
    for off in t.cosets:
        for o in off:
            if (o * 2 ** FIX).denominator != 1 or not (0 <= o <= hi) or (rounding != ROUND_NEAREST and o == 1):
                return False
    amp = 2 ** (FIX - 1) if rounding == ROUND_NEAREST else 2 ** FIX
    for nrm, off in t.planes:
        if any(Fraction(w).denominator != 1 for w in nrm):
            return False
        if (off * 2 ** FIX).denominator != 1 or abs(off) * 2 ** FIX >= 2 ** 31:
            return False
        if sum(abs(int(w)) for w in nrm) * amp >= 2 ** 31:   # |DOT| fits int32
            return False
    for nrm, (b0, r, sc, m1) in plane_families(t).items():
        if sc > 2 ** FIX:
            return False
    return True


# -- expression emission -------------------------------------------------------------


class Emitter:
    def __init__(self, fw: str):
        self.fw = fw
        self.T = "float" if fw == F32 else "double"
        self.lines = []
        self.nt = 0
        self.indent = "  "

    def tmp(self, prefix="t"):
        self.nt += 1
        return f"{prefix}{self.nt}"

    def line(self, text):
        self.lines.append(self.indent + text)

    def tree2(self, node, u, c):
        """Packed (float2) emission of a Horner tree for two queries at once: FFMA2 / FADD2 /
        FMUL2 with broadcast immediates; a product feeding exactly one sum is fused."""
        uses = {}
        stack = [node]
        seen = set()
        while stack:
            nd = stack.pop()
            if id(nd) in seen:
                continue
            seen.add(id(nd))
            if isinstance(nd, (Add, Mul)):
                for ch in (nd.left, nd.right):
                    uses[id(ch)] = uses.get(id(ch), 0) + 1
                    stack.append(ch)
        out = {}
        fused = {}

        def lit(q):
            v = flit(q, F32)
            return f"make_float2({v}, {v})"
        stack = [(node, False)]
        while stack:
            nd, done = stack.pop()
            key = id(nd)
            if key in out:
                continue
            if isinstance(nd, Const):
                out[key] = lit(nd.value)
            elif isinstance(nd, Var):
                out[key] = u[nd.index]
            elif isinstance(nd, Sym):
                out[key] = c[nd.index]
            elif not done:
                stack.append((nd, True))
                if isinstance(nd, Add):
                    # one product used only here is emitted inside the FMA: visit its operands
                    fz = fused.get(key)
                    if fz is None:
                        fz = next((ch for ch in (nd.left, nd.right) if isinstance(ch, Mul)
                                   and uses.get(id(ch), 0) == 1 and id(ch) not in out), False)
                        fused[key] = fz
                    for ch in (nd.right, nd.left):
                        if fz is not False and ch is fz:
                            stack.append((ch.right, False))
                            stack.append((ch.left, False))
                        else:
                            stack.append((ch, False))
                else:
                    stack.append((nd.right, False))
                    stack.append((nd.left, False))
            else:
                t = self.tmp("p")
                if isinstance(nd, Add):
                    l, r = nd.left, nd.right
                    fz = fused.get(key, False)
                    if fz is not False:
                        m, other = (l, r) if fz is l else (r, l)
                        expr = (f"__ffma2_rn({out[id(m.left)]}, {out[id(m.right)]}, "
                                f"{out[id(other)]})")
                    else:
                        expr = f"__fadd2_rn({out[id(l)]}, {out[id(r)]})"
                else:
                    expr = f"__fmul2_rn({out[id(nd.left)]}, {out[id(nd.right)]})"
                self.line(f"const float2 {t} = {expr};")
                out[key] = t
        return out[id(node)]

    def tree(self, node, u, c, consts=None):
        """Post-order emission of a Horner tree; returns the operand string."""
        out = {}
        stack = [(node, False)]
        while stack:
            nd, done = stack.pop()
            key = id(nd)
            if key in out:
                continue
            if isinstance(nd, Const):
                out[key] = consts(nd.value) if consts else flit(nd.value, self.fw)
            elif isinstance(nd, Var):
                out[key] = u[nd.index]
            elif isinstance(nd, Sym):
                out[key] = c[nd.index]
            elif not done:
                stack.append((nd, True))
                stack.append((nd.right, False))
                stack.append((nd.left, False))
            else:
                a, b = out[id(nd.left)], out[id(nd.right)]
                t = self.tmp()
                op = "+" if isinstance(nd, Add) else "*"
                self.line(f"const {self.T} {t} = {a} {op} {b};")
                out[key] = t
        return out[id(node)]


# -- program ----------------------------------------------------------------------


@dataclass
class CudaProgram:
    """A generated kernel: source + the metadata the C ABI needs."""
    name: str
    source: str
    entry: str
    dim: int
    ncosets: int
    float_width: str
    block: int
    halo: int
    extents: tuple           # per coset (unpadded)
    padded_extents: tuple
    has_grad: bool
    has_dbg: bool
    config: GenConfig
    space: SplineSpace = field(repr=False)
    mode: str = "direct"
    bin: int = 0
    brick: tuple = ()
    smem_bytes: int = 0
    chunk: int = 0
    queries_per_thread: int = 1   # sorted mode: tile / block (one CTA tile per grid step)
    presort: int = 0              # bin edge of the C ABI's locality pre-sort (sorted mode)
    stage_tma: bool = False
    rounding: int = 1
    meta: dict = field(default_factory=dict)

    @property
    def key(self) -> str:
        return hashlib.sha256(self.source.encode()).hexdigest()[:24]

    @property
    def dtype(self):
        return np.float32 if self.float_width == F32 else np.float64


DYN_TABLE_MIN = 40 * 1024     # sorted mode: larger shared tables live in dynamic shared memory


def _monomial_chunks(nm: int, tchunk: int):
    """Monomial ranges of the chunked table passes (multiples of 4 wide): one pass up to
    96 monomials (order <= 3 in 3-D), else passes of about `tchunk` (0: 80)."""
    size = tchunk or (nm if nm <= 96 else 80)
    size = max(4, -(-size // 4) * 4)
    return [(m0, min(nm, m0 + size)) for m0 in range(0, nm, size)]


def _sigma_short(t: Tables) -> bool:
    return all(-32768 <= v < 32768 for v in t.sigma)


def _table_bytes(space, t: Tables, cfg) -> int:
    """Upper estimate of the per-CTA shared-memory tables (sigma, transforms, offsets, LUT)."""
    b = 0
    if len(t.sigma) <= cfg.sigma_smem:
        b += (2 if _sigma_short(t) else 4) * len(t.sigma)
    b += 4 * 12 * t.nsub            # transforms + t'
    b += 4 * (t.n + 1) * t.nsub     # stencil offsets (table mode)
    b += 4 * t.nsub                 # psi
    if cfg.coeffs == "table":
        nm = len({e for rp in space.ref_polys for (e, _c) in rp.poly.terms})
        b += 4 * t.K * (t.n + 1) * (-(-nm // 4) * 4)
    return b


def _chunk_trees(space, cfg, t: Tables):
    """Per reference polynomial: per chunk, the tree to evaluate (or None)."""
    m = cfg.params.group_size
    out = []
    for i, rp in enumerate(space.ref_polys):
        cs = group_polynomial(rp.poly, m, range(t.n_psi[i]))
        trees = []
        for poly, block in cs.chunks:
            if not poly:
                trees.append(None)
                continue
            if cfg.form == "horner":
                trees.append(horner_factorize(poly))
            else:
                node = None
                free = Poly(poly.dim, {k: v for k, v in poly.terms.items() if k[1] == NO_SYMBOL})
                if free:
                    node = horner_factorize(free)
                for j in block:
                    w = poly.coefficient_of(j)
                    if not w:
                        continue
                    term = Mul(horner_factorize(w), Sym(j))
                    node = term if node is None else Add(node, term)
                trees.append(node)
        out.append(trees)
    return out


def _grad_trees(space, cfg, t: Tables):
    """Per reference polynomial, per axis: one Horner tree of d psi / d u_axis."""
    out = []
    for rp in space.ref_polys:
        per = []
        for a in range(t.s):
            dp = rp.poly.differentiate(a)
            per.append(horner_factorize(dp) if dp else None)
        out.append(per)
    return out


def generate(space, config: GenConfig | None = None, extents=None,
             validate: bool = True) -> CudaProgram:
    """Generate the CUDA kernel for `space` (reference `generate`, codegen.py:508).

    `extents`: per-coset volume extents (tuple of s ints, or one tuple per coset);
    the kernel is specialized on the padded strides so every fetch offset of a
    uniform stencil is an immediate.  Defaults to 64 per axis.
    """
    if not isinstance(space, SplineSpace):
        space = SplineSpace.adopt(space)
    errors = [d for d in validate_space(space) if d.severity == "error"] if validate else []
    if errors:
        raise ValueError(f"space is not valid: {errors[0]}")
    cfg = config or default_config(space)
    t = derive_tables(space)
    s, M = t.s, t.M
    if extents is None:
        extents = (64,) * s
    ext = tuple(tuple(int(v) for v in e) for e in extents) if isinstance(extents[0], (tuple, list)) \
        else tuple(tuple(int(v) for v in extents) for _ in range(M))
    if len(ext) != M or any(len(e) != s for e in ext):
        raise ValueError(f"extents must give {s} values for each of {M} cosets")
    if cfg.fetch == "linear":
        from .linfetch import generate_linear
        return generate_linear(space, cfg, ext)
    h = t.halo
    binned = cfg.mode == "binned"
    render = cfg.mode == "render"
    # sorted evaluation: mode "sorted", or the renderer with tile > 0 (samples of a block of
    # RB rays x (tile / RB) steps are sorted by psi like queries of a sorted tile)
    sorted_ = cfg.mode == "sorted" or (render and cfg.tile > 0)
    RB = 128   # sorted render: rays per CTA block (four 8 x 4-pixel warp tiles)
    presort = cfg.presort if (sorted_ and not render) else 0
    if cfg.presort and not presort:
        raise ValueError("presort applies to mode='sorted' (query kernels)")
    if presort and (s > 3 or len(set(ext)) != 1):
        raise ValueError("presort needs equal coset extents and dimension <= 3")
    pack2 = cfg.pack == 2
    if pack2:
        if cfg.float_width != F32 or cfg.mode not in ("direct", "binned"):
            raise ValueError("pack=2 supports f32 kernels in direct or binned mode")
        if not (M == 1 or cfg.unroll_cosets) or cfg.coeffs != "imm":
            raise ValueError("pack=2 needs unrolled cosets and immediate coefficients")
        if len(space.ref_polys) > 1 and cfg.params.branch_mode != PREDICATED:
            raise ValueError("pack=2 evaluates every reference polynomial (predicated dispatch)")
    if render and cfg.tile > 0 and (cfg.tile % RB or cfg.block % 32):
        raise ValueError("sorted render: tile must be a multiple of 128 rays")
    if render and (cfg.float_width != F32 or s != 3 or not (M == 1 or cfg.unroll_cosets)):
        raise ValueError("render mode supports f32 kernels of dimension 3 with unrolled cosets")
    if sorted_:
        if cfg.float_width != F32 or s > 3:
            raise ValueError("sorted mode supports f32 kernels of dimension <= 3")
        # per-tile psi counters live in a 32-entry shared array (one warp scans them), and
        # pair keys pack (rank | sub << 16) into an int
        if t.K > 32:
            raise ValueError(f"sorted mode supports at most 32 reference polynomials, not {t.K}")
        if t.nsub >= 1 << 15:
            raise ValueError(f"sorted mode supports fewer than 32768 sub-regions, not {t.nsub}")
        if not cfg.unroll_cosets:
            raise ValueError("sorted mode unrolls the coset loop")
        # per (query, coset) pair: record (u, base) 16 B + order 4 B + key/result 4 B
        # (16 B result with the gradient); two CTAs per SM share the 227 KB
        pair_bytes = 36 if cfg.grad else 24
        if cfg.tile == 0:
            tb = _table_bytes(space, t, cfg)
            # tables beyond the static limit go to dynamic shared memory beside the pair
            # records; then one CTA per SM owns the 227 KB
            room = (110 if tb <= DYN_TABLE_MIN else 210) * 1024 - tb
            tq = max(cfg.block, min(8192, room // (M * pair_bytes)) // cfg.block * cfg.block)
            tq = min(tq, max(cfg.block, 2048 // cfg.block * cfg.block))
            cfg = replace(cfg, tile=tq)
    bin_ = cfg.bin
    rm0 = space.region_map
    if binned:
        if cfg.float_width != F32 or s > 3:
            raise ValueError("binned mode supports f32 kernels of dimension <= 3")
        if rm0.shape == PARALLELEPIPED and not exact.is_identity(rm0.basis):
            raise ValueError("binned mode needs an identity region-of-evaluation basis")
        if len(set(ext)) != 1:
            raise ValueError("binned mode needs equal coset extents")
        if any(not (0 <= c < 1) for off in t.cosets for c in off):
            raise ValueError("binned mode needs coset offsets in [0, 1)")
        margin = h + 2   # f32 binning may be off by one cell; rounding/cosets add one more
        H = margin
        unit = 4  # TMA: innermost box extent x 4 B must be a multiple of 16 B
        tbytes = _table_bytes(space, t, cfg)
        budget = max(16 * 1024, cfg.brick_budget - tbytes)
        if bin_ == 0:   # largest multiple of 4 whose bricks (all cosets) fit the budget
            bin_ = 4
            while M * 4 * (-(-(bin_ + 4 + 2 * margin) // unit) * unit) ** s <= budget \
                    and bin_ + 4 <= max(ext[0]):
                bin_ += 4
        if bin_ % 4:
            raise ValueError("bin must be a multiple of 4 (TMA box coordinates must be 16-B aligned)")
        nb = [-(-e // bin_) for e in ext[0]]
        while int(np.prod(nb)) > 16384:        # the binning kernels' shared histogram limit
            bin_ += 4
            nb = [-(-e // bin_) for e in ext[0]]
        # TMA boxes: every extent a multiple of 4 elements and start coordinates multiples
        # of 4 (measured on sm_100a: other alignments fault), padded extents multiples of 16
        brick = [-(-(bin_ + 2 * margin) // unit) * unit] * s
        prow = [max(ext[0][d] + 2 * H, (nb[d] - 1) * bin_ + brick[d]) for d in range(s)]
        prow = [-(-v // 16) * 16 for v in prow]
        pext = tuple(tuple(prow) for _ in range(M))
        bstr = [1] * s
        for d in range(s - 2, -1, -1):
            bstr[d] = bstr[d + 1] * brick[d + 1]
        brick_elems = bstr[0] * brick[0]
        brick_elems = -(-brick_elems // 32) * 32       # 128-B aligned TMA destinations
        smem_bytes = M * brick_elems * 4
    else:
        H = h
        pext = tuple(tuple(e + 2 * h for e in row) for row in ext)
    for row in pext:
        nel = 1
        for e in row:
            nel *= e
        if nel >= 2 ** 31:
            raise ValueError("coset array too large for 32-bit element offsets")
    strides = []
    for row in pext:
        st = [1] * s
        for d in range(s - 2, -1, -1):
            st[d] = st[d + 1] * row[d + 1]
        strides.append(st)
    same_geom = len(set(pext)) == 1
    smem_fetch = binned and cfg.stage != "l1"
    if smem_fetch:
        strides = [list(bstr) for _ in range(M)]   # fetch offsets are brick-relative
        same_geom = True
    if binned and not smem_fetch:
        smem_bytes = 0

    fw = cfg.float_width
    # query / result streams: evict-first (streaming) so they do not push the coefficient
    # volume out of L2; plain __ldg / stores with stream="default"
    ldf, stf = ("__ldcs", "__stcs") if cfg.stream == "cs" else ("__ldg", "sg_st")
    intsel = cfg.select != "f64" and (M == 1 or cfg.unroll_cosets) and int_selection_ok(space, t, fw)
    if cfg.select == "int" and not intsel:
        raise ValueError("this space/variant cannot use the integer selection path")
    families = plane_families(t)
    em = Emitter(fw)
    T = em.T
    P = t.modulus
    symforms = None
    if cfg.form == "sym":
        from .symmetry import symmetrize
        symforms = []
        for i, rp in enumerate(space.ref_polys):
            sub = next(sb for sb in space.subregions if sb.psi_index == i)
            symforms.append(symmetrize(rp.poly, sub.stencil))
    trees = _chunk_trees(space, cfg if cfg.form != "sym" else replace(cfg, form="horner"), t)
    gtrees = _grad_trees(space, cfg, t) if cfg.grad else None
    if symforms is not None:
        sym_trees = [horner_factorize(f.poly) if f is not None else None for f in symforms]
        sym_gtrees = None
        if cfg.grad:
            sym_gtrees = [[horner_factorize(f.poly.differentiate(a)) if f is not None
                           and f.poly.differentiate(a) else None for a in range(t.s)]
                          if f is not None else None for f in symforms]
    # one (m, d) plan per reference polynomial (codegen.py:332-356); with per-polynomial
    # stencil sizes the plans differ, and a dispatch that evaluates several polynomials on
    # one fetched stencil (predicated) fetches all n sites first
    psi_plans = [schedule_pipeline(group_polynomial(rp.poly, cfg.params.group_size,
                                                    range(t.n_psi[i])), cfg.params)
                 for i, rp in enumerate(space.ref_polys)]
    plan = psi_plans[0]
    # every site of the largest stencil, chunked like a polynomial of n symbols: chunk b of
    # any polynomial only uses symbols of block b, so all of them can follow this plan
    plan_all = plan if t.uniform_n else schedule_pipeline(
        group_polynomial(Poly(s, {}), cfg.params.group_size, range(t.n)), cfg.params)

    def plan_for(psis):
        return psi_plans[psis[0]] if len(psis) == 1 else plan_all
    if t.uniform_n:
        assert all(p.steps == plan.steps for p in psi_plans), "plans differ across sub-regions"
    elif pack2 or cfg.prefetch:
        raise ValueError("pack=2 / prefetch need one stencil size for every sub-region")
    refetch = cfg.params.refetch_tables

    head = []
    A = head.append
    A(f"// generated by paper_2102_08518_b200.cudagen for space '{space.name}'")
    A(f"// m={cfg.params.group_size} d={cfg.params.pipeline_depth} mode={cfg.params.branch_mode} "
      f"refetch={str(refetch).lower()} unroll_cosets={str(cfg.unroll_cosets).lower()} "
      f"form={cfg.form} coeffs={cfg.coeffs} {fw} block={cfg.block} grad={int(cfg.grad)} "
      f"dbg={int(cfg.dbg)}")
    A(f"// extents={ext} stencil reach={h} padded={pext[0]} halo={H} mode={cfg.mode}"
      + (f" bin={bin_} brick={tuple(brick)} stage={cfg.stage}" if binned else "")
      + (f" presort={presort}" if presort else ""))
    A("struct SgCosets { const void* base[8]; };")
    A("template <typename T> __device__ __forceinline__ void sg_st(T* p, T v) { *p = v; }")
    if binned:
        A("struct __align__(64) SgTmap { unsigned long long opaque[16]; };")
        A("struct SgTmaps { SgTmap m[8]; };")

    # ---- tables ------------------------------------------------------------
    smem = []     # (name, ctype, values)
    use_sigma = t.nsub > 1 and len(space.planes) > 0 and len(set(t.sigma)) > 1
    sigma_global = use_sigma and len(t.sigma) > cfg.sigma_smem
    families = plane_families(t)
    # radix: when every plane belongs to a threshold family, the family counts (c_f in
    # 0..r_f) index a table directly -- sub = sigma[(sum_f ((1 << c_f) - 1) << b0_f) mod p]
    # is precomputed for every count combination, so no bit assembly and no modulo remain
    radix = None
    tab_r = []
    if cfg.radix and use_sigma and families:
        fam_planes = sum(r for (_b0, r, _sc, _m1) in families.values())
        combos = 1
        for (_b0, r, _sc, _m1) in families.values():
            combos *= r + 1
        if fam_planes == len(t.planes) and combos <= (1 << 18):
            fl = sorted(families.items(), key=lambda kv: kv[1][0])
            strides_r, acc_ = {}, 1
            for nrm, (b0, r, sc, m1) in reversed(fl):
                strides_r[nrm] = acc_
                acc_ *= r + 1
            for idx in range(combos):
                q, rem = 0, idx
                for nrm, (b0, r, sc, m1) in fl:
                    c_ = (rem // strides_r[nrm]) % (r + 1)
                    q |= ((1 << c_) - 1) << b0
                tab_r.append(t.sigma[q % t.modulus] if (t.compress or q < len(t.sigma)) else -1)
            radix = strides_r
    # sign vectors: 32-bit masks, 64-bit when more than 32 planes cross the cell (an
    # extension of the reference's 32-plane limit, model.validate_space); the radix index
    # is always small
    wide = len(t.planes) > 32 and radix is None
    if len(t.planes) > 64:
        raise ValueError("at most 64 BSP planes")
    QT, QS, QO = ("unsigned long long", "ull", "1ull") if wide else ("unsigned", "u", "1u")
    if use_sigma and not sigma_global and radix is None:
        smem.append(("sg_sigma", "short" if _sigma_short(t) else "int", list(t.sigma)))
    tq = s == 3 and fw == F32 and not (t.uniform_T and t.uniform_tp)
    if tq:
        # rows (T[d][0], T[d][1], T[d][2], t'[d]) per sub-region: 3 LDS.128 per coset
        smem.append(("sg_Tq", T, [float(v) for tr, tp in zip(t.transforms, t.tshift)
                                  for d in range(3) for v in (*tr[d], tp[d])]))
    else:
        if not t.uniform_T:
            smem.append(("sg_T", T, [float(v) for tr in t.transforms for row in tr for v in row]))
        if not t.uniform_tp:
            smem.append(("sg_tp", T, [float(v) for tp in t.tshift for v in tp]))
    fetch_mode = "uniform" if t.uniform_stencil else ("affine" if t.affine is not None else "table")
    if (fetch_mode == "table" and t.paffine is not None and sorted_ and cfg.coeffs != "table"
            and cfg.fetch_offsets == "affine"):
        # sorted dispatch evaluates one reference polynomial per arm, so its fetch offsets
        # can be boff + sum_e m_j[e] sp_e with the polynomial's own reference stencil m as
        # compile-time constants: one int4 load per pair instead of one (bank-conflicted)
        # table load per stencil site
        fetch_mode = "paffine"
    if cfg.tloop:
        fetch_mode = "table"      # the site loop reads its offsets from the per-sub-region table
    if fetch_mode != "uniform" and not same_geom and not cfg.unroll_cosets:
        pass  # per-coset strides are compile-time constants in unrolled mode only; handled below
    if fetch_mode in ("affine", "paffine"):
        # per geometry g: S'_sub = A_sub^T S (s ints) and boff_sub = b_sub . S
        for g, st in enumerate(strides if not same_geom else strides[:1]):
            vals = []
            for A_, b_ in (t.affine if fetch_mode == "affine" else t.paffine):
                sp = [sum(A_[d][e] * st[d] for d in range(s)) for e in range(s)]
                vals += sp + [sum(b_[d] * st[d] for d in range(s))]
            smem.append((f"sg_aff{g}", "int", vals))
    elif fetch_mode == "table":
        npad = t.n + 1 if t.n % 2 == 0 else t.n
        for g, st in enumerate(strides if not same_geom else strides[:1]):
            vals = []
            for sten in t.stencils:
                row = [sum(site[d] * st[d] for d in range(s)) for site in sten]
                vals += row + [0] * (npad - len(row))
            smem.append((f"sg_off{g}", "int", vals))
    if not t.uniform_psi and t.K > 1:
        smem.append(("sg_psi", "int", list(t.psi)))
    tab = None
    if cfg.coeffs == "table":
        # monomial-major lookup table: A[psi][j][m] = coefficient of u^e_m c_j in psi
        exps = sorted({e for rp in space.ref_polys for (e, _c) in rp.poly.terms})
        nm = len(exps)
        nmp = -(-nm // 4) * 4
        midx = {e: i for i, e in enumerate(exps)}
        # layout [site j][monomial quad q][psi][4]: for a fixed (j, q) the threads of a
        # warp read consecutive 16-B chunks indexed by their own psi -> the LDS.128s are
        # bank-conflict free (distinct psi) or broadcasts (equal psi), and the (j, q)
        # offset is an immediate
        w4 = 4 if T == "float" else 2
        nq = nmp // w4
        Atab = [0.0] * (t.n * nq * t.K * w4)
        A0tab = [0.0] * (t.K * nmp)
        for k_, rp in enumerate(space.ref_polys):
            for (e, c), q in rp.poly.terms.items():
                if c == NO_SYMBOL:
                    A0tab[k_ * nmp + midx[e]] = q
                else:
                    mi = midx[e]
                    Atab[((c * nq + mi // w4) * t.K + k_) * w4 + mi % w4] = q
        tab = dict(exps=exps, nm=nm, nmp=nmp, nq=nq,
                   has_free=any(v != 0 for v in A0tab))
        smem.append(("sg_A", T, Atab))
        if tab["has_free"]:
            smem.append(("sg_A0", T, A0tab))
        if 4 * len(Atab) > (190 if sorted_ else 96) * 1024:
            raise ValueError("coefficient table too large for shared memory")
        if not t.uniform_n:
            smem.append(("sg_npsi", "int", list(t.n_psi)))

    lut = []
    if cfg.coeffs == "lut":
        lut_index = {}

        def lut_const(q):
            v = float(np.float32(float(q))) if fw == F32 else float(q)
            if v not in lut_index:
                lut_index[v] = len(lut)
                lut.append(v)
            return f"sg_lut[{lut_index[v]}]"
        consts = lut_const
    else:
        consts = None

    for name, ctype, vals in smem:
        lit = ", ".join(repr(v) if ctype not in ("int", "short") else str(v) for v in vals)
        if ctype == "float":
            lit = ", ".join(flit(Fraction(v), F32) for v in vals)
        elif ctype == "double":
            lit = ", ".join(dlit(Fraction(v)) for v in vals)
        # global (not __constant__): the per-CTA staging copy reads thread-distinct addresses,
        # which the constant cache serializes; coalesced __ldg reads do not
        A(f"__device__ const __align__(16) {ctype} {name}_c[{len(vals)}] = {{{lit}}};")
    gset = {g for g in cfg.gtables.split(",") if g}
    if gset:
        if cfg.mode == "binned":
            raise ValueError("gtables applies to the sorted / direct / render kernels")
        bad = sorted(g for g in gset if not g.startswith("sg_"))
        if bad:   # tables a space does not have (e.g. sg_psi with one polynomial) are skipped
            raise ValueError(f"gtables: {bad} are not shared-table names (sg_Tq, sg_aff0, ...)")
    gtabs = [e for e in smem if e[0] in gset]
    smem = [e for e in smem if e[0] not in gset]

    if radix is not None:
        A(f"__device__ const short sg_sigma_r[{len(tab_r)}] = {{{', '.join(str(v) for v in tab_r)}}};")
    if sigma_global and radix is None:
        A(f"__device__ const int sg_sigma_g[{len(t.sigma)}] = {{{', '.join(str(v) for v in t.sigma)}}};")

    # sorted mode: shared tables beyond the static limit go to dynamic shared memory, after
    # the tile's pair records (offsets fixed here; sorted_smem adds their bytes)
    dyn_tables, dyn_bytes = {}, 0
    if sorted_:
        elem = {"float": 4, "double": 8, "int": 4, "short": 2}
        static_b = sum(elem[ct] * len(v) for _n, ct, v in smem)
        if static_b > DYN_TABLE_MIN:
            pair_b = M * cfg.tile * (36 if cfg.grad else 24) + (cfg.tile * 4 if presort else 0)
            off = -(-pair_b // 16) * 16
            for name, ct, v in sorted(smem, key=lambda e: -elem[e[1]] * len(e[2])):
                if static_b <= DYN_TABLE_MIN // 4:
                    break
                nb = elem[ct] * len(v)
                dyn_tables[name] = (ct, off)
                off += -(-nb // 16) * 16
                static_b -= nb
            dyn_bytes = off - -(-pair_b // 16) * 16 + (-(-pair_b // 16) * 16 - pair_b)

    if not sorted_:
        elem = {"float": 4, "double": 8, "int": 4, "short": 2}
        static_b = sum(elem[ct] * len(v) for _n, ct, v in smem)
        if static_b > 46 * 1024:
            raise ValueError(f"shared tables of {static_b} B exceed the 48 KB static limit "
                             "(only mode='sorted' places large tables in dynamic shared memory)")

    # ---- kernel -------------------------------------------------------------
    def direct_preamble(pre="  "):
        """Per query (direct mode): the query point from xs[qi] + the fixed-point split."""
        out = []
        for d in range(s):
            if intsel:
                out.append(f"{pre}const float xq{d} = {ldf}(&xs[qi * {s} + {d}]);")
                out.append(f"{pre}const double x{d} = (double)xq{d};")
            else:
                out.append(f"{pre}const double x{d} = (double){ldf}(&xs[qi * {s} + {d}]);")
        if intsel:
            out.extend(pre + ln for ln in int_prelude())
        return out

    def binned_preamble(pre="  "):
        """Per query (binned mode, record q4 in scope): original index, point, fixed-point
        split, and the coset-0 shift relative to the (approximately assigned) bin:
        loc = k + rel lands in [0, brick) for every coset and stencil site."""
        out = []
        Q = out.append
        Q(f"{pre}const long long qi = (long long)__float_as_int(q4.w);")
        comps = ["x", "y", "z"]
        for d in range(s):
            if intsel:
                Q(f"{pre}const float xq{d} = q4.{comps[d]};")
            Q(f"{pre}const double x{d} = (double)q4.{comps[d]};")
        if intsel:
            out.extend(pre + ln for ln in int_prelude())
        rnd0 = rm0.rounding if rm0.shape == PARALLELEPIPED else ROUND_NEAREST

        def kb_f64(p2):
            for d in range(s):
                if rnd0 == ROUND_NEAREST:
                    Q(f"{p2}kb{d} = __double2ll_rz(__dadd_rn(x{d}, copysign(0.5, x{d})));")
                else:
                    Q(f"{p2}kb{d} = __double2ll_rd(x{d});")
                e_ = ext[0][d]
                Q(f"{p2}kbw{d} = (int)kb{d};")
                Q(f"{p2}if ((unsigned)kbw{d} >= {e_}u) {{ long long m_ = kb{d} % {e_}LL; kbw{d} = (int)(m_ < 0 ? m_ + {e_}LL : m_); }}")
        for d in range(s):
            Q(f"{pre}long long kb{d}; int kbw{d};")
        if intsel:
            # fast range (2^-7 <= x < E): the coset-0 shift in fixed point, 0 <= kb <= E
            Q(f"{pre}if (fast_) {{")
            for d in range(s):
                e_ = ext[0][d]
                C = (1 << (FIX - 1)) if rnd0 == ROUND_NEAREST else 0
                Q(f"{pre}  const int kq{d} = hi{d}_ + ((lo{d}_ + {C}) >> 30);")
                Q(f"{pre}  kb{d} = kq{d}; kbw{d} = kq{d} >= {e_} ? kq{d} - {e_} : kq{d};")
            Q(f"{pre}}} else {{")
            kb_f64(pre + "  ")
            Q(f"{pre}}}")
        else:
            kb_f64(pre)
        for d in range(s):
            e_ = ext[0][d]
            Q(f"{pre}int u{d}_ = kbw{d} - lo{d};")
            Q(f"{pre}if (u{d}_ < -1) u{d}_ += {e_}; else if (u{d}_ > {bin_}) u{d}_ -= {e_};")
            Q(f"{pre}const long long rel{d} = (long long)(u{d}_ + {margin}) - kb{d};")
        return out

    def int_prelude():
        """Per query: fixed-point split x = hi + lo * 2^-30 (lo in [0, 2^30)), exact for the
        fast-path range 2^-7 <= x < E (so 0 <= k <= E: one conditional subtract wraps it);
        other queries take the fp64 path."""
        emin = [min(e[d] for e in ext) for d in range(s)]
        out = ["const bool fast_ = " + " && ".join(
            f"(xq{d} >= 0x1p-7f) && (xq{d} < {float(emin[d])!r}f)" for d in range(s)) + ";"]
        for d in range(s):
            out.append(f"const long long X{d}_ = __float2ll_rn(xq{d} * 0x1p+30f);")
            out.append(f"const int hi{d}_ = (int)(X{d}_ >> 30);")
            out.append(f"const int lo{d}_ = (int)X{d}_ & 0x3fffffff;")
        return out

    # sorted: 2 CTAs / SM by design; render: an explicit bound (ptxas otherwise caps at 48 regs)
    min_blocks = cfg.min_blocks or ((1 if (dyn_tables or cfg.tpairs == 2) else 2) if sorted_
                                    else (max(1, 256 // cfg.block) if (render or pack2) else 0))
    lb = f"{cfg.block}, {min_blocks}" if min_blocks else f"{cfg.block}"
    body = []
    B = body.append
    if not binned:
        B(f'extern "C" __global__ void __launch_bounds__({lb}) {ENTRY}(')
        if render:
            # fused volume renderer: one ray per thread, `steps` samples,
            # reconstruction (+ gradient shading) and front-to-back compositing in registers
            B("    const float4* __restrict__ rays, long long n, float4* __restrict__ rgba,")
            B("    const float* __restrict__ tf, int steps, unsigned* __restrict__ err, SgCosets vol) {")
        else:
            B(f"    const {T}* __restrict__ xs, long long n, {T}* __restrict__ out, {T}* __restrict__ grad,")
            B("    int* __restrict__ dbg, unsigned* __restrict__ err, SgCosets vol) {")
        for name, ctype, vals in smem:
            if name not in dyn_tables:
                B(f"  __shared__ __align__(16) {ctype} {name}[{len(vals)}];")
        if sorted_:
            B("  extern __shared__ __align__(16) unsigned char sg_dyn[];")
            for name, (ctype, off) in dyn_tables.items():
                B(f"  {ctype}* {name} = reinterpret_cast<{ctype}*>(sg_dyn + {off});")
        for name, ctype, vals in smem:
            B(f"  for (int i_ = threadIdx.x; i_ < {len(vals)}; i_ += {cfg.block}) {name}[i_] = __ldg(&{name}_c[i_]);")
        for name, ctype, _vals in gtabs:
            B(f"  const {ctype}* __restrict__ {name} = {name}_c;")
        if sorted_:
            TQ = cfg.tile
            MP = M * TQ
            B("  float4* sg_rec = reinterpret_cast<float4*>(sg_dyn);")
            # the pair keys (rank | sub << 16) live in the result array until the scatter
            if cfg.grad:
                B(f"  float4* sg_res4 = reinterpret_cast<float4*>(sg_dyn + {MP * 16});")
                B(f"  int* sg_key = reinterpret_cast<int*>(sg_dyn + {MP * 16});")
                B(f"  int* sg_ord = reinterpret_cast<int*>(sg_dyn + {MP * 32});")
            else:
                B(f"  float* sg_res = reinterpret_cast<float*>(sg_dyn + {MP * 16});")
                B(f"  int* sg_key = reinterpret_cast<int*>(sg_dyn + {MP * 16});")
                B(f"  int* sg_ord = reinterpret_cast<int*>(sg_dyn + {MP * 20});")
            B("  __shared__ int sg_cnt[32];")
            B("  __shared__ int sg_start[32];")
            B("  __shared__ int sg_tot;")
            if cfg.cmajor == 3:
                B("  __shared__ int sg_next;")
            B("  if (threadIdx.x < 32) sg_cnt[threadIdx.x] = 0;")
            B("  const unsigned lane = threadIdx.x & 31u;")
            B("  const unsigned lt_mask = (1u << lane) - 1u;")
            for l in range(M):
                B(f"  const int coff{l} = (int)((const float*)vol.base[{l}] - (const float*)vol.base[0]);")
            B("  __syncthreads();")
            sorted_smem = MP * pair_bytes + (TQ * 4 if presort else 0) + dyn_bytes
            if presort:
                # original index of every tile query (the input is the locality-sorted records)
                B(f"  int* sg_qidx = reinterpret_cast<int*>(sg_dyn + {MP * pair_bytes});")
            ind = "  "
            if render:
                B(f"  const float tf_lo = tf[0], tf_inv = tf[1], tf_op = tf[2];")
                B("  const float c0lo = tf[3], c1lo = tf[4], c2lo = tf[5];")
                B("  const float c0d = tf[6] - tf[3], c1d = tf[7] - tf[4], c2d = tf[8] - tf[5];")
                if cfg.grad:
                    B("  const float L0 = tf[9], L1 = tf[10], L2 = tf[11];")
                # persistent ray blocks; each block marches its RB rays in chunks of SJ steps
                B("  __shared__ long long sg_rb0;")
                B("  for (;;) {   // ray blocks claimed in order from the per-launch counter err[1]")
                B(f"  if (threadIdx.x == 0) sg_rb0 = (long long)atomicAdd(err + 1, 1u) * {RB};")
                B("  __syncthreads();")
                B("  const long long rb0 = sg_rb0;")
                B("  if (rb0 >= n) break;")
                B(f"  const long long myray = rb0 + threadIdx.x;")
                B(f"  float my_dt = 0.f;")
                B(f"  if (threadIdx.x < {RB} && myray < n) my_dt = __ldg(&rays[2 * myray + 1]).w;")
                B("  const float my_aop = tf_op * my_dt;")
                B("  float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;")
                B(f"  for (int j0 = 0; j0 < steps; j0 += {TQ // RB}) {{")
            else:
                # persistent tiles: the shared tables are staged once per CTA
                # tiles are claimed in order from a per-launch counter (err[1], zeroed by the
                # C ABI before the launch): the resident CTAs work on a contiguous window of
                # the query stream -- coherent L1/L2 footprint, no tail imbalance
                B("  __shared__ long long sg_q0;")
                if cfg.cflip:
                    B("  int sg_par = 1;")
                B("  for (;;) {")
                B(f"  if (threadIdx.x == 0) sg_q0 = (long long)atomicAdd(err + 1, 1u) * {TQ};")
                B("  __syncthreads();")
                B("  const long long q0 = sg_q0;")
                B("  if (q0 >= n) break;")
                if cfg.cflip:
                    B("  sg_par ^= 1;")
        elif smem:
            B("  __syncthreads();")
        if sorted_:
            pass
        elif render:
            B(f"  const float tf_lo = tf[0], tf_inv = tf[1], tf_op = tf[2];")
            B("  const float c0lo = tf[3], c1lo = tf[4], c2lo = tf[5];")
            B("  const float c0d = tf[6] - tf[3], c1d = tf[7] - tf[4], c2d = tf[8] - tf[5];")
            if cfg.grad:
                B("  const float L0 = tf[9], L1 = tf[10], L2 = tf[11];")
            B(f"  for (long long qi = (long long)blockIdx.x * {cfg.block} + threadIdx.x; qi < n;")
            B(f"       qi += (long long)gridDim.x * {cfg.block}) {{")
            B("  const float4 ra = __ldg(&rays[2 * qi]), rb = __ldg(&rays[2 * qi + 1]);")
            B("  const float o0 = ra.x, o1 = ra.y, o2 = ra.z, r0 = ra.w, r1 = rb.x, r2 = rb.y;")
            B("  const float t0 = rb.z, rdt = rb.w;")
            B("  const float aop = tf_op * rdt;")
            B("  float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;")
            B("  #pragma unroll 1")
            B("  for (int j = 0; j < steps; ++j) {")
            # sample positions in round-to-nearest fp32 ops (no contraction): the oracle
            # forms the same float32 expression
            B("  const float tj = __fadd_rn(t0, __fmul_rn(__fadd_rn((float)j, 0.5f), rdt));")
            for d in range(s):
                B(f"  const float xq{d} = __fadd_rn(o{d}, __fmul_rn(tj, r{d}));")
                B(f"  const double x{d} = (double)xq{d};")
            if intsel:
                body.extend("  " + ln for ln in int_prelude())
            ind = "  "
        else:
          # grid-stride loop: the shared tables are staged once per CTA, not once per 128 queries
          if pack2:
              B(f"  for (long long q0_ = (long long)blockIdx.x * {2 * cfg.block}; q0_ < n;")
              B(f"       q0_ += (long long)gridDim.x * {2 * cfg.block}) {{")
          else:
              B(f"  for (long long qi = (long long)blockIdx.x * {cfg.block} + threadIdx.x; qi < n;")
              B(f"       qi += (long long)gridDim.x * {cfg.block}) {{")
              body.extend(direct_preamble())
          ind = "  "
    else:
        B(f'extern "C" __global__ void __launch_bounds__({lb}) {ENTRY}(')
        B("    const float4* __restrict__ sorted, const int* __restrict__ starts,")
        B("    const int2* __restrict__ items,")
        B(f"    {T}* __restrict__ out, {T}* __restrict__ grad, int* __restrict__ dbg,")
        B("    unsigned* __restrict__ err, SgCosets vol, const __grid_constant__ SgTmaps tm) {")
        B("  extern __shared__ __align__(128) float sg_brick[];")
        B("  __shared__ __align__(8) unsigned long long sg_bar;")
        for name, ctype, vals in smem:
            B(f"  __shared__ __align__(16) {ctype} {name}[{len(vals)}];")
        # work item of this CTA: (bin, first sorted query); bin < 0 -> no work
        B("  const int2 item = items[blockIdx.x];")
        B("  if (item.x < 0) return;")
        B("  const int bin = item.x;")
        rem = "bin"
        for d in range(s - 1, -1, -1):
            if d == 0:
                B(f"  const int lo0 = ({rem}) * {bin_};")
            else:
                B(f"  const int lo{d} = (({rem}) % {nb[d]}) * {bin_};")
                rem = f"({rem}) / {nb[d]}"
        gst = [1] * s
        for d in range(s - 2, -1, -1):
            gst[d] = gst[d + 1] * pext[0][d + 1]
        if cfg.stage == "l1":
            pass
        elif cfg.stage == "tma":
            coords = ", ".join(f"%{2 + i}" for i in range(s))
            cvals = ", ".join(f'"r"(lo{d})' for d in range(s - 1, -1, -1))
            B("  const unsigned sg_bar_a = (unsigned)__cvta_generic_to_shared(&sg_bar);")
            B("  if (threadIdx.x == 0) {")
            B('    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sg_bar_a) : "memory");')
            B('    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");')
            B('    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");')
            box_bytes = 4
            for e in brick:
                box_bytes *= e
            B(f'    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sg_bar_a), "r"({M * box_bytes}) : "memory");')
            for l in range(M):
                B(f"    {{ const unsigned dst = (unsigned)__cvta_generic_to_shared(sg_brick + {l * brick_elems});")
                B(f'      asm volatile("cp.async.bulk.tensor.{s}d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {{{coords}}}], [%{2 + s}];"')
                B(f'                   :: "r"(dst), "l"((unsigned long long)&tm.m[{l}]), {cvals}, "r"(sg_bar_a) : "memory"); }}')
            B("  }")
        else:
            bz = brick[-1]
            box_elems = 1
            for e in brick:
                box_elems *= e
            for l in range(M):
                off0 = sum(H * gst[d] for d in range(s))
                B(f"  {{ const float* __restrict__ G = (const float*)vol.base[{l}] - {off0};")
                B(f"    for (int e_ = threadIdx.x; e_ < {box_elems}; e_ += {cfg.block}) {{")
                idx = []
                r_ = "e_"
                for d in range(s - 1, -1, -1):
                    if d == 0:
                        idx.insert(0, f"({r_})")
                    else:
                        idx.insert(0, f"(({r_}) % {brick[d]})")
                        r_ = f"({r_}) / {brick[d]}"
                addr = " + ".join(f"(lo{d} + {idx[d]}) * {gst[d]}" for d in range(s))
                B(f"      sg_brick[{l * brick_elems} + e_] = __ldg(G + {addr}); }} }}")
        for name, ctype, vals in smem:
            B(f"  for (int i_ = threadIdx.x; i_ < {len(vals)}; i_ += {cfg.block}) {name}[i_] = __ldg(&{name}_c[i_]);")
        B("  __syncthreads();")
        if cfg.stage == "tma" and smem_fetch:
            B('  asm volatile("{\\n .reg .pred p;\\n SG_WAIT_%=:\\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\\n @!p bra SG_WAIT_%=;\\n}" :: "r"(sg_bar_a) : "memory");')
        B(f"  const int q_end = min(starts[bin + 1], item.y + {cfg.chunk});")
        if pack2:
            B(f"  for (int qq = item.y + threadIdx.x; qq < q_end; qq += {2 * cfg.block}) {{")
        else:
            B("  int qq = item.y + threadIdx.x;")
            B(f"  float4 q4n = qq < q_end ? {ldf}(&sorted[qq]) : make_float4(0.f, 0.f, 0.f, 0.f);")
            B(f"  for (; qq < q_end; qq += {cfg.block}) {{")
            B("  const float4 q4 = q4n;")
            B(f"  if (qq + {cfg.block} < q_end) q4n = {ldf}(&sorted[qq + {cfg.block}]);   // prefetch the next record")
            body.extend(binned_preamble())
        ind = "  "
    if not sorted_ and not pack2:
        B(f"{ind}{T} acc = ({T})0;")
        if cfg.grad:
            for d in range(s):
                B(f"{ind}{T} gacc{d} = ({T})0;")
    em.lines = []
    sctx = {}

    def emit_sorted_record(l, emit_u):
        """Sorted mode, phase 1: store the (query, coset) pair's record and take its
        rank within its psi class (warp-aggregated shared-memory counter)."""
        L = em.line
        for d in range(s):
            L(f"const float xf{d} = {f'xff{d}' if intsel else f'(float)xc{d}'};")
        us = emit_u("") + ["0.0f"] * (3 - s)
        if t.K > 1:
            L(f"const int psi_ = {t.psi[0] if t.uniform_psi else 'sg_psi[sub]'};")
        else:
            L("const int psi_ = 0;")
        L(f"sg_rec[{l * sctx['TQ']} + ql] = make_float4({us[0]}, {us[1]}, {us[2]}, "
          f"__int_as_float(base + coff{l}));")
        if cfg.rank == "atomic":
            # one shared-memory atomic per pair (same-class lanes serialize in the unit)
            L(f"const int rk_ = valid ? atomicAdd(&sg_cnt[psi_], 1) : 0;")
            L(f"sg_key[{l * sctx['TQ']} + ql] = valid ? (rk_ | (sub << 16)) : -1;")
            return
        L(f"const int kp_ = valid ? psi_ : {t.K};")
        L("const unsigned mm_ = __match_any_sync(0xffffffffu, kp_);")
        L("const int ld_ = __ffs(mm_) - 1;")
        L("int rb_ = 0;")
        L(f"if ((int)lane == ld_ && kp_ < {t.K}) rb_ = atomicAdd(&sg_cnt[kp_], __popc(mm_));")
        L("rb_ = __shfl_sync(0xffffffffu, rb_, ld_);")
        L(f"sg_key[{l * sctx['TQ']} + ql] = valid ? ((rb_ + __popc(mm_ & lt_mask)) | (sub << 16)) : -1;")

    def emit_u_factory(L):
        """u = T_sub x_loc + t'_sub from the xf{d} (f32/f64 x_loc) in scope."""

        def emit_u(tag):
            us = []
            if tq:
                for d in range(3):
                    L(f"const float4 tq{d}{tag} = *reinterpret_cast<const float4*>(&sg_Tq[sub * 12 + {4 * d}]);")
                    name = f"u{d}{tag}"
                    L(f"const float {name} = tq{d}{tag}.x * xf0 + tq{d}{tag}.y * xf1 + "
                      f"tq{d}{tag}.z * xf2 + tq{d}{tag}.w;")
                    us.append(name)
                return us
            for d in range(s):
                if t.uniform_T:
                    row = t.transforms[0][d]
                    acc = None
                    for e in range(s):
                        w = row[e]
                        if w == 0:
                            continue
                        term = f"xf{e}" if w == 1 else (f"(-xf{e})" if w == -1
                                                         else f"{flit(w, fw)} * xf{e}")
                        acc = term if acc is None else f"{acc} + {term}"
                    acc = acc or f"({T})0"
                else:
                    acc = " + ".join(f"sg_T[sub * {s * s} + {d * s + e}] * xf{e}" for e in range(s))
                if t.uniform_tp:
                    tp = t.tshift[0][d]
                    if tp != 0:
                        acc = f"{acc} + {flit(tp, fw)}"
                else:
                    acc = f"{acc} + sg_tp[sub * {s} + {d}]"
                name = f"u{d}{tag}"
                L(f"const {T} {name} = {acc};")
                us.append(name)
            return us
        return emit_u

    def emit_int_select(l, rounding, wrap_ext=None):
        """Fixed-point rho + plane bits for coset l (assigns kk{d}, xff{d}, qq).

        x = hi + lo 2^-30, o = O 2^-30.  round half away (x >= 2^-7, o <= 1/2: the value
        x - o is never a negative tie): k = hi + ((lo - O + 2^29) >> 30),
        x_loc = ((lo - O + 2^29) & (2^30 - 1)) - 2^29.  floor: k = hi + ((lo - O) >> 30),
        x_loc = (lo - O) & (2^30 - 1).  Plane dots are exact int32 sums; a family's count
        is floor(dot 2^p) = DOT >> (30 - p)."""
        L = em.line
        for d in range(s):
            O = int(t.cosets[l][d] * 2 ** FIX)
            if rounding == ROUND_NEAREST:
                C = (1 << (FIX - 1)) - O
                L(f"const int t{d}_ = lo{d}_ + ({C});" if C else f"const int t{d}_ = lo{d}_;")
                L(f"const int k{d}_ = hi{d}_ + (t{d}_ >> 30);")
                L(f"kk{d} = (long long)k{d}_;")
                if wrap_ext:
                    L(f"kwv{d} = k{d}_ >= {wrap_ext[d]} ? k{d}_ - {wrap_ext[d]} : k{d}_;")
                L(f"const int xc{d}_ = (t{d}_ & 0x3fffffff) - 0x20000000;")
            else:
                L(f"const int t{d}_ = lo{d}_ - ({O});" if O else f"const int t{d}_ = lo{d}_;")
                L(f"const int k{d}_ = hi{d}_ + (t{d}_ >> 30);")
                L(f"kk{d} = (long long)k{d}_;")
                if wrap_ext:
                    L(f"kwv{d} = k{d}_ < 0 ? k{d}_ + {wrap_ext[d]} : k{d}_;")
                L(f"const int xc{d}_ = t{d}_ & 0x3fffffff;")
            L(f"xff{d} = (float)xc{d}_ * 0x1p-30f;")
        if not space.planes:
            return
        idots = {}

        def idot(nrm):
            if nrm not in idots:
                terms = []
                for e in range(s):
                    w = int(nrm[e])
                    if w == 0:
                        continue
                    terms.append((w, f"xc{e}_"))
                expr = ""
                for w, v in terms:
                    mag = f"{v}" if abs(w) == 1 else f"{abs(w)} * {v}"
                    expr += (f" + {mag}" if w > 0 else f" - {mag}") if expr else (mag if w > 0 else f"-{mag}")
                idots[nrm] = f"di{len(idots)}_"
                L(f"const int {idots[nrm]} = {expr or '0'};")
            return idots[nrm]
        done = set()
        for i, (nrm, off) in enumerate(t.planes):
            if nrm in families:
                if nrm in done:
                    continue
                done.add(nrm)
                b0, r, sc, m1 = families[nrm]
                sh = FIX - (sc.bit_length() - 1)
                dv = idot(nrm)
                cnt = em.tmp("cnt")
                arg = f"({dv} >> {sh}) - ({m1 - 1})" if m1 != 1 else f"{dv} >> {sh}"
                L(f"const int {cnt} = min(max({arg}, 0), {r});")
                if radix is not None:
                    L(f"qq += (unsigned)({cnt} * {radix[nrm]});")
                else:
                    L(f"qq |= (({QO} << {cnt}) - {QO}) << {b0};")
                continue
            D = int(off * 2 ** FIX)
            L(f"qq |= ({idot(nrm)} >= {D}) ? {1 << i}{QS} : 0{QS};")

    def emit_coset(l, dyn, phase="all"):
        """Body for coset `l` (int) or the loop variable `l` (dyn=True).

        phase "all": selection, fetch and evaluation inline (direct / binned modes).
        Sorted mode splits it: "select" emits the selection and stores the pair's
        record (u, flat base index) and its rank within its psi class; "eval" emits
        fetch + evaluation for a record whose sub, base, u0.. and psi are in scope."""
        L = em.line if phase != "eval" else (lambda text: None)
        dguard = "if (valid) " if phase == "select" else ""
        if dyn:
            if smem_fetch:
                L(f"const float* V = sg_brick + l * {brick_elems};")
            else:
                ptr = f"(const {T}*)vol.base[0]"
                for c in range(1, M):
                    ptr = f"(l == {c} ? (const {T}*)vol.base[{c}] : {ptr})"
                L(f"const {T}* __restrict__ V = {ptr};")
        else:
            if smem_fetch:
                L(f"const float* V = sg_brick + {l * brick_elems};")
            else:
                L(f"const {T}* __restrict__ V = (const {T}*)vol.base[{l}];")
        rm = space.region_map
        if rm.shape == PARALLELEPIPED:
            basis, rounding = rm.basis, rm.rounding
        else:
            basis, rounding = exact.eye(s), ROUND_NEAREST
        isel = intsel and not dyn and phase != "eval"
        wrap_ext = list(ext[0 if same_geom else l]) if (isel and not smem_fetch) else None
        if isel:
            # fast path: exact 2^-30 fixed point (int32); the fp64 path below handles the
            # queries outside [2^-7, E) (tiny, negative, beyond the box) bit-identically
            for d in range(s):
                L(f"long long kk{d}; float xff{d};" + (f" int kwv{d};" if wrap_ext else ""))
            L(f"{QT} qq = 0{QS};")
            L("if (fast_) {")
            em.indent += "  "
            emit_int_select(l, rounding, wrap_ext)
            em.indent = em.indent[:-2]
            L("} else {")
            em.indent += "  "
        if dyn:
            for d in range(s):
                offs = [float(t.cosets[c][d]) for c in range(M)]
                if all(o == 0.0 for o in offs):
                    L(f"const double xl{d} = x{d};")
                else:
                    expr = dlit(t.cosets[0][d])
                    for c in range(1, M):
                        expr = f"(l == {c} ? {dlit(t.cosets[c][d])} : {expr})"
                    L(f"const double xl{d} = __dsub_rn(x{d}, {expr});")
        else:
            for d in range(s):
                o = t.cosets[l][d]
                if o == 0:
                    L(f"const double xl{d} = x{d};")
                else:
                    L(f"const double xl{d} = __dsub_rn(x{d}, {dlit(o)});")
        # ---- rho (codegen.py:190-226, oracle.py:38-53)

        def rnd(v):
            # round half away from zero == trunc(v + copysign(1/2, v)) with the same RN
            # addition the oracle performs (floor(v+1/2) / ceil(v-1/2), oracle.py:34-35);
            # converted to an integer in one cvt.rzi / cvt.rmi
            if rounding == ROUND_NEAREST:
                return f"__double2ll_rz(__dadd_rn(({v}), copysign(0.5, ({v}))))"
            return f"__double2ll_rd({v})"
        if exact.is_identity(basis):
            for d in range(s):
                L(f"const long long k{d} = {rnd(f'xl{d}')};")
        else:
            inv = exact.inverse(basis)
            for d in range(s):
                acc = None
                for e in range(s):
                    if inv[d][e] == 0:
                        continue
                    term = f"xl{e}" if inv[d][e] == 1 else f"__dmul_rn(xl{e}, {dlit(inv[d][e])})"
                    acc = term if acc is None else f"__dadd_rn({acc}, {term})"
                L(f"const double bu{d} = {acc or '0.0'};")
                L(f"const long long r{d} = {rnd(f'bu{d}')};")
            for d in range(s):
                terms = [f"{int(basis[d][e])}LL * r{e}" for e in range(s) if basis[d][e] != 0]
                L(f"const long long k{d} = {' + '.join(terms) or '0LL'};")
        for d in range(s):
            L(f"const double xc{d} = __dsub_rn(xl{d}, (double)k{d});")
        # ---- membership (codegen.py:230-250; oracle dot = left-to-right)
        if space.planes:
            L(f"{QT} q = 0{QS};")
            dots = {}   # one fp64 dot product per distinct normal (planes share families)
            fam_done = set()
            counted = families
            for i, (nrm, off) in enumerate(t.planes):
                if nrm in counted:
                    if nrm in fam_done:
                        continue
                    fam_done.add(nrm)
                    acc = None
                    for e in range(s):
                        w = nrm[e]
                        if w == 0:
                            continue
                        term = f"xc{e}" if w == 1 else (f"(-xc{e})" if w == -1
                                                          else f"__dmul_rn(xc{e}, {dlit(w)})")
                        acc = term if acc is None else f"__dadd_rn({acc}, {term})"
                    b0, r, sc, m1 = counted[nrm]
                    cnt = em.tmp("cnt")
                    L(f"const int {cnt} = min(max(__double2int_rd(({acc or '0.0'}) * {float(sc)!r}) - ({m1 - 1}), 0), {r});")
                    if radix is not None:
                        L(f"q += (unsigned)({cnt} * {radix[nrm]});")
                    else:
                        L(f"q |= (({QO} << {cnt}) - {QO}) << {b0};")
                    continue
                nz = [(e, w) for e, w in enumerate(nrm) if w != 0]
                if off == 0 and len(nz) == 2 and all(abs(w) == 1 for _, w in nz):
                    # a.x >= 0 with two unit coefficients is an exact comparison:
                    # RN(xa +- xb) >= 0  <=>  xa >= -+xb (sign of an IEEE sum is exact)
                    (ea, wa), (eb, wb) = nz
                    lhs = f"xc{ea}" if wa == 1 else f"(-xc{ea})"
                    rhs = f"(-xc{eb})" if wb == 1 else f"xc{eb}"
                    L(f"q |= ({lhs} >= {rhs}) ? {1 << i}{QS} : 0{QS};")
                    continue
                if nrm not in dots:
                    acc = None
                    for e in range(s):
                        w = nrm[e]
                        if w == 0:
                            continue
                        term = f"xc{e}" if w == 1 else (f"(-xc{e})" if w == -1
                                                          else f"__dmul_rn(xc{e}, {dlit(w)})")
                        acc = term if acc is None else f"__dadd_rn({acc}, {term})"
                    dots[nrm] = f"dn{len(dots)}"
                    L(f"const double {dots[nrm]} = {acc or '0.0'};")
                L(f"q |= ({dots[nrm]} >= {dlit(off)}) ? {1 << i}{QS} : 0{QS};")
        if isel:
            for d in range(s):
                L(f"kk{d} = k{d}; xff{d} = (float)xc{d};")
                if wrap_ext:
                    L(f"kwv{d} = (int)k{d};")
                    L(f"if ((unsigned)kwv{d} >= {wrap_ext[d]}u) {{ long long m_ = k{d} % {wrap_ext[d]}LL; "
                      f"kwv{d} = (int)(m_ < 0 ? m_ + {wrap_ext[d]}LL : m_); }}")
            if space.planes:
                L("qq = q;")
            em.indent = em.indent[:-2]
            L("}")
            for d in range(s):
                L(f"const long long k{d} = kk{d};")
            if space.planes:
                L(f"{QT} q = qq;")
        if space.planes:
            if radix is not None:
                L("int sub = __ldg(&sg_sigma_r[q]);")
            elif t.compress:
                L(f"q = q % {P}{QS};")
            if radix is not None:
                pass
            elif sigma_global:
                L("int sub = __ldg(&sg_sigma_g[q]);")
            elif use_sigma:
                L("int sub = sg_sigma[q];")
            else:
                v = t.sigma[0] if t.sigma else 0
                L(f"int sub = {v};")
            if any(x < 0 for x in t.sigma):
                if use_sigma:
                    L("if (sub < 0) { atomicOr(err, 1u); sub = 0; }")
                else:
                    bad = [qq for qq, x in enumerate(t.sigma) if x < 0]
                    cond = " || ".join(f"q == {qq}{QS}" for qq in bad)
                    L(f"if ({cond}) atomicOr(err, 1u);")
        else:
            L("const int sub = 0;")
        if cfg.dbg:
            cols = s + 1
            base = f"(qi * {M} + {l}) * {cols}" if not dyn else f"(qi * {M} + l) * {cols}"
            for d in range(s):
                L(f"{dguard}dbg[{base} + {d}] = (int)k{d};")
            L(f"{dguard}dbg[{base} + {s}] = sub;")
        # ---- wrap k once per coset, flat base index in the padded array
        geo = 0 if (same_geom or dyn) else l
        if not same_geom and dyn:
            raise ValueError("rolled coset loop needs equal coset extents")
        e_ = ext[geo]
        st_ = strides[geo]
        if smem_fetch:
            for d in range(s):
                L(f"const int kw{d} = (int)(k{d} + rel{d});")
        elif wrap_ext:
            for d in range(s):
                L(f"const int kw{d} = kwv{d};")
        else:
            for d in range(s):
                L(f"int kw{d} = (int)k{d};")
                L(f"if ((unsigned)kw{d} >= {e_[d]}u) {{ long long m_ = k{d} % {e_[d]}LL; "
                  f"kw{d} = (int)(m_ < 0 ? m_ + {e_[d]}LL : m_); }}")
        L("const int base = " + " + ".join(
            f"kw{d} * {st_[d]}" if st_[d] != 1 else f"kw{d}" for d in range(s)) + ";")
        if phase == "select":
            emit_sorted_record(l, emit_u_factory(L))
            return
        L = em.line
        # ---- per-sub fetch offsets
        if fetch_mode == "paffine":
            gi = 0 if same_geom else geo
            if s == 3:
                L(f"const int4 aff = *reinterpret_cast<const int4*>(&sg_aff{gi}[sub * 4]);")
                for e, comp in zip(range(3), "xyz"):
                    L(f"const int sp{e} = aff.{comp};")
                L("const int boff = base + aff.w;")
            else:
                L(f"const int* aff = &sg_aff{gi}[sub * {s + 1}];")
                for e in range(s):
                    L(f"const int sp{e} = aff[{e}];")
                L(f"const int boff = base + aff[{s}];")

            def off_expr(j):
                site = t.ref_psi[sctx["cur_psi"]][j]
                parts = ["boff"]
                for e in range(s):
                    v = site[e]
                    if v == 1:
                        parts.append(f"sp{e}")
                    elif v == -1:
                        parts.append(f"-sp{e}")
                    elif v:
                        parts.append(f"{v} * sp{e}")
                return " + ".join(parts).replace("+ -", "- ")
        elif fetch_mode == "affine":
            gi = 0 if same_geom else geo
            if s == 3:
                L(f"const int4 aff = *reinterpret_cast<const int4*>(&sg_aff{gi}[sub * 4]);")
                for e, comp in zip(range(3), "xyz"):
                    L(f"const int sp{e} = aff.{comp};")
                L("const int boff = base + aff.w;")
            else:
                L(f"const int* aff = &sg_aff{gi}[sub * {s + 1}];")
                for e in range(s):
                    L(f"const int sp{e} = aff[{e}];")
                L(f"const int boff = base + aff[{s}];")
            vals = {e: sorted({site[e] for site in t.ref_stencil}) for e in range(s)}
            for e in range(s):
                for v in vals[e]:
                    if v == 0:
                        continue
                    name = f"mp{e}_{v}" if v > 0 else f"mn{e}_{-v}"
                    L(f"const int {name} = {v} * sp{e};")

            def off_expr(j):
                site = t.ref_stencil[j]
                parts = ["boff"]
                for e in range(s):
                    v = site[e]
                    if v:
                        parts.append(f"mp{e}_{v}" if v > 0 else f"mn{e}_{-v}")
                return " + ".join(parts)
        elif fetch_mode == "table":
            gi = 0 if same_geom else geo
            npad = t.n + 1 if t.n % 2 == 0 else t.n
            L(f"const int* offt = &sg_off{gi}[sub * {npad}];")

            def off_expr(j):
                return f"base + offt[{j}]"
        else:
            sten = t.stencils[0]

            def off_expr(j):
                o = sum(sten[j][d] * st_[d] for d in range(s))
                return f"base + ({o})" if o else "base"
        if phase == "gather":
            # pack=2: this query's u, coefficients, psi (and sub) go to outer variables
            q = sctx["q"]
            for d in range(s):
                L(f"const {T} xf{d} = {f'xff{d}' if (intsel and not dyn) else f'({T})xc{d}'};")
            for j in range(t.n):
                if smem_fetch:
                    L(f"const float c{j} = V[{off_expr(j)}];")
                else:
                    L(f"const float c{j} = __ldg(V + ({off_expr(j)}));")
            us = emit_u_factory(L)("")
            for d in range(s):
                L(f"pu{q}{l}_{d} = {us[d]};")
            for j in range(t.n):
                L(f"pc{q}{l}_{j} = c{j};")
            if t.K > 1:
                L(f"ps{q}{l} = {t.psi[0] if t.uniform_psi else 'sg_psi[sub]'};")
            if cfg.grad:
                L(f"sb{q}{l} = sub;")
            return
        # ---- local point u = T x_loc + t'
        if phase == "all":
            for d in range(s):
                L(f"const {T} xf{d} = {f'xff{d}' if (intsel and not dyn) else f'({T})xc{d}'};")

        def emit_u(tag):
            if phase == "eval":
                return [f"u{d}" for d in range(s)]     # loaded from the pair's record
            return emit_u_factory(L)(tag)

        # ---- fetch + compute following the (m, d) plan
        if t.K > 1 and phase != "eval":
            if t.uniform_psi:
                L(f"const int psi = {t.psi[0]};")
            else:
                L("const int psi = sg_psi[sub];")
        cvars = [f"c{j}" for j in range(t.n)]

        def fetch_line(j, tag):
            if phase == "eval" and sctx.get("prefetched"):
                return f"const {T} c{j}{tag} = pfc{j};"     # loaded one iteration ahead
            if smem_fetch:
                return f"const {T} c{j}{tag} = V[{off_expr(j)}];"
            return f"const {T} c{j}{tag} = __ldg(V + ({off_expr(j)}));"

        def run_plan_sym(psis, tag):
            """All fetches in plan order, then per psi the symmetry-mixed symbols and
            one Horner evaluation of psi'(v, s) (form "sym")."""
            for step in plan_for(psis).steps:
                if step.kind == FETCH:
                    j = step.index
                    L(fetch_line(j, tag))
            u = emit_u(tag)
            accs, grads = {}, ({} if cfg.grad else None)
            for i in psis:
                f = symforms[i]
                cv = [f"c{j}{tag}" for j in range(t.n)]
                if f is None:
                    v = em.tree(horner_factorize(space.ref_polys[i].poly), u, cv, consts)
                    accs[i] = v
                    if cfg.grad:
                        grads[i] = [em.tree(gtrees[i][a], u, cv, consts) if gtrees[i][a] is not None
                                    else f"({T})0" for a in range(s)]
                    continue
                vv = []
                for d in range(s):
                    if f.shift[d] != 0:
                        nm = em.tmp("v")
                        L(f"const {T} {nm} = {u[d]} - {flit(f.shift[d], fw)};")
                        vv.append(nm)
                    else:
                        vv.append(u[d])
                sv = [None] * len(f.mixes)
                kk = len(f.axes)
                for reps, syms in f.orbits:
                    if len(reps) == 1 << kk:
                        # free orbit: fast Walsh-Hadamard butterflies over the flip group
                        x = {bits: cv[j] for bits, j in reps}
                        for tb in range(kk):
                            nx = {}
                            for b in x:
                                if b >> tb & 1:
                                    continue
                                hi = b | (1 << tb)
                                a_, b_ = em.tmp("w"), em.tmp("w")
                                L(f"const {T} {a_} = {x[b]} + {x[hi]};")
                                L(f"const {T} {b_} = {x[b]} - {x[hi]};")
                                nx[b], nx[hi] = a_, b_
                            x = nx
                        for P, k_ in syms.items():
                            sv[k_] = x[P]
                    else:
                        for P, k_ in syms.items():
                            expr = ""
                            for sign, j in f.mixes[k_]:
                                expr += (" + " if sign > 0 else " - ") + cv[j] if expr else (
                                    cv[j] if sign > 0 else f"-{cv[j]}")
                            nm = em.tmp("s")
                            L(f"const {T} {nm} = {expr};")
                            sv[k_] = nm
                accs[i] = em.tree(sym_trees[i], vv, sv, consts)
                if cfg.grad:
                    grads[i] = [em.tree(sym_gtrees[i][a], vv, sv, consts)
                                if sym_gtrees[i][a] is not None else f"({T})0" for a in range(s)]
            return accs, grads, u

        def run_plan(psis, tag):
            if symforms is not None:
                return run_plan_sym(psis, tag)
            accs = {i: None for i in psis}
            u = None
            nchunk = 0
            for step in plan_for(psis).steps:
                if step.kind == FETCH:
                    j = step.index
                    L(fetch_line(j, tag))
                elif step.kind == COMPUTE:
                    if u is None or refetch:
                        u = emit_u(f"{tag}_{nchunk}" if refetch else tag)
                    for i in psis:
                        if step.index >= len(trees[i]):
                            continue
                        tree = trees[i][step.index]
                        if tree is None:
                            continue
                        cv = [f"{c}{tag}" for c in cvars]
                        v = em.tree(tree, u, cv, consts)
                        if accs[i] is None:
                            accs[i] = v
                        else:
                            nt = em.tmp("a")
                            L(f"const {T} {nt} = {accs[i]} + {v};")
                            accs[i] = nt
                    nchunk += 1
            grads = None
            if cfg.grad:
                grads = {}
                for i in psis:
                    cv = [f"{c}{tag}" for c in cvars]
                    du = []
                    for a in range(s):
                        tr = gtrees[i][a]
                        du.append(em.tree(tr, u, cv, consts) if tr is not None else f"({T})0")
                    grads[i] = du
            return {i: (v if v is not None else f"({T})0") for i, v in accs.items()}, grads, u

        def add_grad(du, tr_known):
            # grad_x += T^T du  (T = sub transform)
            for e in range(s):
                parts = []
                for a in range(s):
                    if t.uniform_T:
                        w = t.transforms[0][a][e]
                        if w == 0:
                            continue
                        parts.append(du[a] if w == 1 else (f"(-{du[a]})" if w == -1
                                                           else f"{flit(w, fw)} * {du[a]}"))
                    else:
                        if tq:
                            parts.append(f"sg_Tq[sub * 12 + {4 * a + e}] * {du[a]}")
                        else:
                            parts.append(f"sg_T[sub * {s * s} + {a * s + e}] * {du[a]}")
                if parts:
                    L(f"gacc{e} += {' + '.join(parts)};")

        def nested_horner(coef, u, exps=None):
            """sum_e coef(e) u^e over the exponent set (default tab['exps']) by nested
            Horner (axis 0 outermost).  coef(e) returns an operand string or None."""
            exps = tab["exps"] if exps is None else exps

            def rec(fixed, axis):
                if axis == s:
                    return coef(tuple(fixed))
                pows = sorted({e[axis] for e in exps if tuple(e[:axis]) == tuple(fixed)})
                if not pows:
                    return None
                r = None
                for a in range(pows[-1], -1, -1):
                    q = rec(list(fixed) + [a], axis + 1) if a in pows else None
                    if r is None:
                        r = q
                    else:
                        nt = em.tmp("h")
                        if q is None:
                            L(f"const {T} {nt} = {r} * {u[axis]};")
                        else:
                            L(f"const {T} {nt} = {r} * {u[axis]} + {q};")
                        r = nt
                return r
            return rec([], 0) or f"({T})0"

        def run_table():
            nmp = tab["nmp"]
            midx = {e: i for i, e in enumerate(tab["exps"])}
            psi_e = "psi" if t.K > 1 else "0"
            vec = "float4" if T == "float" else "double2"
            w = 4 if T == "float" else 2
            comps = ["x", "y", "z", "w"][:w]
            L(f"const {vec}* __restrict__ Arow = reinterpret_cast<const {vec}*>(sg_A) + {psi_e};")
            if sctx.get("dual"):
                return run_table_dual(nmp, midx, psi_e, vec, w, comps)
            mchunks = _monomial_chunks(tab["nm"], cfg.tchunk) if cfg.tloop else [(0, tab["nm"])]
            if len(mchunks) > 1:
                return run_table_chunked(nmp, midx, psi_e, vec, w, comps, mchunks)
            for m in range(nmp):
                L(f"{T} g{m} = ({T})0;")
            u = None
            nchunk = 0
            if cfg.tloop:
                # one runtime loop over the polynomial's stencil sites: the same few hundred
                # instructions serve every reference polynomial (large K x n tables would
                # otherwise be unrolled into per-polynomial code that thrashes the I-cache);
                # the next site's coefficient is fetched one iteration ahead
                if fetch_mode != "table":
                    raise ValueError("tloop needs per-sub-region offset tables")
                nsite = (f"sg_npsi[{psi_e}]" if not t.uniform_n else str(t.n))
                L(f"const int ns_ = {nsite};")
                rd = (lambda o: f"V[{o}]") if smem_fetch else (lambda o: f"__ldg(V + ({o}))")
                L(f"{T} cn_ = {rd('base + offt[0]')};")
                L("#pragma unroll 1")
                L("for (int j_ = 0; j_ < ns_; ++j_) {")
                L(f"  const {T} cj_ = cn_;")
                L(f"  if (j_ + 1 < ns_) cn_ = {rd('base + offt[j_ + 1]')};")
                L(f"  const {vec}* __restrict__ Aj_ = Arow + j_ * {tab['nq'] * t.K};")
                for q in range(nmp // w):
                    L(f"  {{ const {vec} a_ = Aj_[{q * t.K}]; " + " ".join(
                        f"g{q * w + r} = a_.{comps[r]} * cj_ + g{q * w + r};" for r in range(w)) + " }")
                L("}")
            for step in (() if cfg.tloop else plan_all.steps):
                if step.kind == FETCH:
                    j = step.index
                    L(fetch_line(j, ""))
                elif step.kind == COMPUTE:
                    for j in plan_all.blocks[step.index]:
                        for q in range(nmp // w):
                            L(f"{{ const {vec} a_ = Arow[{(j * tab['nq'] + q) * t.K}]; " + " ".join(
                                f"g{q * w + r} = a_.{comps[r]} * c{j} + g{q * w + r};" for r in range(w)) + " }")
                    nchunk += 1
            table_tail(nmp, midx, psi_e)

        def run_table_dual(nmp, midx, psi_e, vec, w, comps):
            """Sorted mode, two pairs A, B of one reference polynomial per thread: every
            coefficient quad read from shared memory feeds 8 FMAs (4 per pair) -- the
            single-pair loop is bound by the shared-memory pipe (one LDS.128 per 4 FMAs)."""
            npad = t.n + 1 if t.n % 2 == 0 else t.n
            L(f"const int* __restrict__ offA_ = &sg_off0[subA * {npad}];")
            L(f"const int* __restrict__ offB_ = &sg_off0[subB * {npad}];")
            for m in range(nmp):
                L(f"{T} gA{m} = ({T})0, gB{m} = ({T})0;")
            nsite = (f"sg_npsi[{psi_e}]" if not t.uniform_n else str(t.n))
            L(f"const int ns_ = {nsite};")
            L(f"{T} cnA_ = __ldg(V + (baseA + offA_[0])), cnB_ = __ldg(V + (baseB + offB_[0]));")
            L("#pragma unroll 1")
            L("for (int j_ = 0; j_ < ns_; ++j_) {")
            L(f"  const {T} cjA_ = cnA_, cjB_ = cnB_;")
            L("  if (j_ + 1 < ns_) { cnA_ = __ldg(V + (baseA + offA_[j_ + 1])); "
              "cnB_ = __ldg(V + (baseB + offB_[j_ + 1])); }")
            L(f"  const {vec}* __restrict__ Aj_ = Arow + j_ * {tab['nq'] * t.K};")
            for q in range(nmp // w):
                L(f"  {{ const {vec} a_ = Aj_[{q * t.K}]; " + " ".join(
                    f"gA{q * w + r} = a_.{comps[r]} * cjA_ + gA{q * w + r}; "
                    f"gB{q * w + r} = a_.{comps[r]} * cjB_ + gB{q * w + r};" for r in range(w)) + " }")
            L("}")
            for tag in "AB":
                L("{")
                em.indent += "  "
                L(f"const int sub = sub{tag};")
                for d in range(s):
                    L(f"const {T} u{d} = u{tag}{d};")
                for m in range(nmp):
                    L(f"{T} g{m} = g{tag}{m};")
                L(f"{T} acc = ({T})0;")
                if cfg.grad:
                    for d in range(s):
                        L(f"{T} gacc{d} = ({T})0;")
                table_tail(nmp, midx, psi_e)
                if cfg.grad:
                    gg = ", ".join([f"gacc{d}" for d in range(s)] + ["0.0f"] * (3 - s))
                    L(f"sg_res4[pi{tag}] = make_float4(acc, {gg});")
                else:
                    L(f"sg_res[pi{tag}] = acc;")
                em.indent = em.indent[:-2]
                L("}")

        def run_table_chunked(nmp, midx, psi_e, vec, w, comps, mchunks):
            """Site loop in passes over monomial ranges [m0, m1): each pass accumulates its
            g_m over every site (the coefficient gathers of later passes hit L1) and folds
            them into the value (+ gradient) by nested Horner over its own monomials, so
            only m1 - m0 accumulators are live -- degree-9 pieces have 220 monomials."""
            u = emit_u("")
            nsite = (f"sg_npsi[{psi_e}]" if not t.uniform_n else str(t.n))
            L(f"const int ns_ = {nsite};")
            for m0, m1 in mchunks:
                L("{")
                em.indent += "  "
                for m in range(m0, -(-m1 // w) * w):
                    L(f"{T} g{m} = ({T})0;")
                L(f"{T} cn_ = __ldg(V + (base + offt[0]));")
                L("#pragma unroll 1")
                L("for (int j_ = 0; j_ < ns_; ++j_) {")
                L(f"  const {T} cj_ = cn_;")
                L("  if (j_ + 1 < ns_) cn_ = __ldg(V + (base + offt[j_ + 1]));")
                L(f"  const {vec}* __restrict__ Aj_ = Arow + j_ * {tab['nq'] * t.K};")
                for q in range(m0 // w, -(-m1 // w)):
                    L(f"  {{ const {vec} a_ = Aj_[{q * t.K}]; " + " ".join(
                        f"g{q * w + r} = a_.{comps[r]} * cj_ + g{q * w + r};" for r in range(w)) + " }")
                L("}")
                table_tail(nmp, midx, psi_e, u=u, exps=tab["exps"][m0:m1], free=(m0 == 0))
                em.indent = em.indent[:-2]
                L("}")

        def table_tail(nmp, midx, psi_e, u=None, exps=None, free=True):
            """acc (+ gacc) from the monomial coefficients g{m} in scope (all monomials, or
            the subset `exps` of one chunked pass)."""
            exps = tab["exps"] if exps is None else list(exps)
            eset = set(exps)
            if tab["has_free"] and free:
                L(f"const {T}* __restrict__ A0row = &sg_A0[{psi_e} * {nmp}];")
                for m in range(tab["nm"]):
                    L(f"g{m} += A0row[{m}];")
            u = emit_u("") if u is None else u
            val = nested_horner(lambda e: f"g{midx[e]}" if e in eset else None, u, exps)
            L(f"acc += {val};")
            if cfg.grad:
                du = []
                for a in range(s):
                    def dcoef(e, a=a):
                        e2 = tuple(v + (k == a) for k, v in enumerate(e))
                        if e2 not in eset:
                            return None
                        f = e[a] + 1
                        return f"g{midx[e2]}" if f == 1 else f"{flit(f, fw)} * g{midx[e2]}"
                    dexps = sorted({tuple(v - (k == a) for k, v in enumerate(e))
                                    for e in exps if e[a] > 0})
                    du.append(nested_horner(dcoef, u, dexps) if dexps else f"({T})0")
                add_grad(du, True)

        if cfg.coeffs == "table":
            run_table()
        elif phase == "eval" and t.K > 1:
            # pairs are sorted by psi: every warp but the class-boundary ones takes one arm
            L("switch (psi) {")
            for i in range(t.K):
                L(f"{'default' if i == t.K - 1 else f'case {i}'}: {{")
                em.indent += "  "
                sctx["cur_psi"] = i
                accs, grads, _ = run_plan([i], f"_{i}")
                L(f"acc += {accs[i]};")
                if cfg.grad:
                    add_grad(grads[i], True)
                em.indent = em.indent[:-2]
                L("} break;")
            L("}")
        elif t.K == 1:
            sctx["cur_psi"] = 0
            accs, grads, _ = run_plan([0], "")
            L(f"acc += {accs[0]};")
            if cfg.grad:
                add_grad(grads[0], True)
        elif cfg.params.branch_mode == PREDICATED:
            accs, grads, _ = run_plan(list(range(t.K)), "")
            sel = " + ".join(f"(psi == {i} ? {accs[i]} : ({T})0)" for i in range(t.K))
            L(f"acc += {sel};")
            if cfg.grad:
                du = []
                for a in range(s):
                    du.append(em.tmp("gd"))
                    L(f"const {T} {du[-1]} = " + " + ".join(
                        f"(psi == {i} ? {grads[i][a]} : ({T})0)" for i in range(t.K)) + ";")
                add_grad(du, True)
        else:  # branchy: compare chain, one arm per reference polynomial
            for i in range(t.K):
                kw = "if" if i == 0 else "} else if"
                cond = f"psi == {i}" if i < t.K - 1 else "true"
                L(f"{kw} ({cond}) {{" if i < t.K - 1 else "} else {")
                em.indent += "  "
                accs, grads, _ = run_plan([i], f"_{i}")
                L(f"acc += {accs[i]};")
                if cfg.grad:
                    add_grad(grads[i], True)
                em.indent = em.indent[:-2]
            L("}")

    def neg2(x):
        return f"make_float2(-({x}).x, -({x}).y)"

    def pair_value(i, U, C, want_grad):
        """(value pair, [grad pairs]) of reference polynomial i, packed float2 (FFMA2) for
        pack=2 (two queries per thread)."""
        L = em.line
        f = symforms[i] if symforms is not None else None
        if f is None:
            if symforms is not None:
                node_list = [horner_factorize(space.ref_polys[i].poly)]
            else:
                node_list = [tr for tr in trees[i] if tr is not None]
            val = None
            for nd in node_list:
                v = em.tree2(nd, U, C)
                if val is None:
                    val = v
                else:
                    nt = em.tmp("p")
                    L(f"const float2 {nt} = __fadd2_rn({val}, {v});")
                    val = nt
            val = val or "make_float2(0.f, 0.f)"
            gr = None
            if want_grad:
                gr = [em.tree2(gtrees[i][a], U, C) if gtrees[i][a] is not None
                      else "make_float2(0.f, 0.f)" for a in range(s)]
            return val, gr
        vv = []
        for d in range(s):
            if f.shift[d] != 0:
                nm = em.tmp("p")
                z = flit(-f.shift[d], F32)
                L(f"const float2 {nm} = __fadd2_rn({U[d]}, make_float2({z}, {z}));")
                vv.append(nm)
            else:
                vv.append(U[d])
        sv = [None] * len(f.mixes)
        kk = len(f.axes)
        for reps, syms in f.orbits:
            if len(reps) == 1 << kk:
                x = {bits: C[j] for bits, j in reps}
                for tb in range(kk):
                    nx = {}
                    for b in x:
                        if b >> tb & 1:
                            continue
                        hi_ = b | (1 << tb)
                        a_, b_ = em.tmp("p"), em.tmp("p")
                        L(f"const float2 {a_} = __fadd2_rn({x[b]}, {x[hi_]});")
                        L(f"const float2 {b_} = __fadd2_rn({x[b]}, {neg2(x[hi_])});")
                        nx[b], nx[hi_] = a_, b_
                    x = nx
                for P, k_ in syms.items():
                    sv[k_] = x[P]
            else:
                for P, k_ in syms.items():
                    expr = None
                    for sign, j in f.mixes[k_]:
                        term = C[j] if sign > 0 else neg2(C[j])
                        if expr is None:
                            expr = term
                        else:
                            nm = em.tmp("p")
                            L(f"const float2 {nm} = __fadd2_rn({expr}, {term});")
                            expr = nm
                    sv[k_] = expr
        val = em.tree2(sym_trees[i], vv, sv)
        gr = None
        if want_grad:
            gr = [em.tree2(sym_gtrees[i][a], vv, sv) if sym_gtrees[i][a] is not None
                  else "make_float2(0.f, 0.f)" for a in range(s)]
        return val, gr

    def emit_pack2_body():
        """pack=2: two queries per thread.  Selection, fetch and u stay scalar per query
        (in their own scopes); the polynomial evaluation runs once on float2 pairs, so
        every FMA / add / mul of the (dominant) polynomial work is one FFMA2 / FADD2 /
        FMUL2 for both queries."""
        Bk = cfg.block
        P_ = body.append
        for q in "AB":
            P_(f"  long long qo{q};")
            for l in range(M):
                P_("  float " + ", ".join(f"pu{q}{l}_{d}" for d in range(s)) + ";")
                P_("  float " + ", ".join(f"pc{q}{l}_{j}" for j in range(t.n)) + ";")
                if t.K > 1:
                    P_(f"  int ps{q}{l};")
                if cfg.grad:
                    P_(f"  int sb{q}{l};")
        for q, off in (("A", 0), ("B", Bk)):
            P_(f"  {{  // query {q}")
            if binned:
                P_(f"    const int qv = qq + {off};")
                P_("    const bool valid = qv < q_end;")
                P_(f"    const float4 q4 = {ldf}(&sorted[valid ? qv : qq]);")
                body.extend(binned_preamble("    "))
            else:
                P_(f"    const long long qraw = q0_ + threadIdx.x + {off};")
                P_("    const bool valid = qraw < n;")
                P_("    const long long qi = valid ? qraw : n - 1;")
                body.extend(direct_preamble("    "))
            P_(f"    qo{q} = valid ? qi : -1;")
            sctx["q"] = q
            for l in range(M):
                em.lines = []
                em.indent = "    "
                em.line(f"{{  // coset {l}")
                em.indent = "      "
                emit_coset(l, False, phase="gather")
                em.indent = "    "
                em.line("}")
                body.extend(em.lines)
            P_("  }")
        P_("  float accA = 0.f, accB = 0.f;")
        if cfg.grad:
            P_("  " + "; ".join(f"float gA{d} = 0.f, gB{d} = 0.f" for d in range(s)) + ";")
        em.lines = []
        em.indent = "  "
        L = em.line

        for l in range(M):
            L(f"{{  // coset {l} (packed)")
            U = []
            for d in range(s):
                L(f"const float2 U{d} = make_float2(puA{l}_{d}, puB{l}_{d});")
                U.append(f"U{d}")
            C = []
            for j in range(t.n):
                L(f"const float2 C{j} = make_float2(pcA{l}_{j}, pcB{l}_{j});")
                C.append(f"C{j}")
            psis = [0] if t.K == 1 else list(range(t.K))
            dsum = {q: [None] * s for q in "AB"}
            for i in psis:
                val, gr = pair_value(i, U, C, cfg.grad)
                for q, comp in (("A", "x"), ("B", "y")):
                    if t.K == 1:
                        L(f"acc{q} += ({val}).{comp};")
                    else:
                        L(f"acc{q} += (ps{q}{l} == {i}) ? ({val}).{comp} : 0.f;")
                    if cfg.grad:
                        for a in range(s):
                            e = f"({gr[a]}).{comp}"
                            if t.K > 1:
                                e = f"((ps{q}{l} == {i}) ? {e} : 0.f)"
                            dsum[q][a] = e if dsum[q][a] is None else f"{dsum[q][a]} + {e}"
            if cfg.grad:
                # grad_x += T_sub^T du per query
                for q in "AB":
                    du = []
                    for a in range(s):
                        nm = em.tmp("d")
                        L(f"const float {nm} = {dsum[q][a]};")
                        du.append(nm)
                    for e in range(s):
                        parts = []
                        for a in range(s):
                            if t.uniform_T:
                                w = t.transforms[0][a][e]
                                if w == 0:
                                    continue
                                parts.append(du[a] if w == 1 else (f"(-{du[a]})" if w == -1
                                                                   else f"{flit(w, F32)} * {du[a]}"))
                            elif tq:
                                parts.append(f"sg_Tq[sb{q}{l} * 12 + {4 * a + e}] * {du[a]}")
                            else:
                                parts.append(f"sg_T[sb{q}{l} * {s * s} + {a * s + e}] * {du[a]}")
                        if parts:
                            L(f"g{q}{e} += {' + '.join(parts)};")
            L("}")
        body.extend(em.lines)
        for q in "AB":
            P_(f"  if (qo{q} >= 0) {{")
            P_(f"    {stf}(&out[qo{q}], acc{q});")
            if cfg.grad:
                for d in range(s):
                    P_(f"    {stf}(&grad[qo{q} * {s} + {d}], g{q}{d});")
            P_("  }")
        P_("  }")   # pair loop
        if binned:
            pass
        P_("}")

    if sorted_:
        TQ, Bk = cfg.tile, cfg.block
        PQ = TQ // Bk
        sctx["TQ"] = TQ
        hoist = cfg.qhoist and not render
        if hoist:
            # every query load of this thread's share of the tile is issued before the first
            # selection: one memory latency per tile instead of one per query
            for r in range(PQ):
                if presort:
                    body.append(f"    const float4 hq{r}_ = {ldf}(reinterpret_cast<const float4*>(xs) + "
                                f"min(q0 + {r * Bk} + (long long)threadIdx.x, n - 1));")
                else:
                    for d in range(s):
                        body.append(f"    const float hq{r}_{d} = {ldf}(&xs[min(q0 + {r * Bk} + "
                                    f"(long long)threadIdx.x, n - 1) * {s} + {d}]);")
        for r in range(PQ):
            body.append(f"    {{  // query {r} of this thread in the tile")
            body.append(f"    const int ql = {r * Bk} + (int)threadIdx.x;")
            if render:
                # sample (ray rb0 + ql % RB, step j0 + ql / RB): positions as in the unsorted
                # renderer (round-to-nearest fp32 ops)
                body.append(f"    const long long ray_ = rb0 + (ql % {RB});")
                body.append(f"    const int j_ = j0 + ql / {RB};")
                body.append("    const bool valid = ray_ < n && j_ < steps;")
                body.append("    const long long rc_ = ray_ < n ? ray_ : n - 1;")
                body.append("    const float4 ra = __ldg(&rays[2 * rc_]), rb = __ldg(&rays[2 * rc_ + 1]);")
                body.append("    const float tj = __fadd_rn(rb.z, __fmul_rn(__fadd_rn((float)j_, 0.5f), rb.w));")
                for d, (oc, dc) in enumerate((("ra.x", "ra.w"), ("ra.y", "rb.x"), ("ra.z", "rb.y"))):
                    body.append(f"    const float xq{d} = __fadd_rn({oc}, __fmul_rn(tj, {dc}));")
                    body.append(f"    const double x{d} = (double)xq{d};")
            elif presort:
                # records (x, y, z, original index) in locality order: the tile's queries are
                # spatially close, so the coefficient gathers stay in L1/L2
                body.append("    const long long qs_ = q0 + ql;")
                body.append("    const bool valid = qs_ < n;")
                if hoist:
                    body.append(f"    const float4 r4_ = hq{r}_;")
                else:
                    body.append(f"    const float4 r4_ = {ldf}(reinterpret_cast<const float4*>(xs) + (valid ? qs_ : n - 1));")
                body.append("    const long long qi = (long long)__float_as_int(r4_.w);")
                body.append("    if (valid) sg_qidx[ql] = (int)qi;")
                for d in range(s):
                    body.append(f"    const float xq{d} = r4_.{'xyz'[d]};")
                    body.append(f"    const double x{d} = (double)xq{d};")
            else:
                body.append("    const long long qi = q0 + ql;")
                body.append("    const bool valid = qi < n;")
                body.append("    const long long qc = valid ? qi : n - 1;")
            for d in range(s if not (render or presort) else 0):
                ld_ = f"hq{r}_{d}" if hoist else f"{ldf}(&xs[qc * {s} + {d}])"
                if intsel:
                    body.append(f"    const float xq{d} = {ld_};")
                    body.append(f"    const double x{d} = (double)xq{d};")
                else:
                    body.append(f"    const double x{d} = (double){ld_};")
            if intsel:
                body.extend("    " + ln for ln in int_prelude())
            sctx["r"] = r
            for l in range(M):
                em.lines = []
                em.indent = "      "
                em.line(f"{{  // coset {l}")
                em.indent = "        "
                emit_coset(l, False, phase="select")
                em.indent = "      "
                em.line("}")
                body.extend(em.lines)
            body.append("    }")
        body.append("    __syncthreads();")
        # exclusive scan of the per-psi counts (K <= 32), counters reset for the next tile
        body.append("    if (threadIdx.x < 32) {")
        body.append(f"      const int c_ = (int)lane < {t.K} ? sg_cnt[lane] : 0;")
        body.append("      int v_ = c_;")
        body.append("      for (int o_ = 1; o_ < 32; o_ <<= 1) { const int w_ = __shfl_up_sync(0xffffffffu, v_, o_); if ((int)lane >= o_) v_ += w_; }")
        body.append("      sg_start[lane] = v_ - c_;")
        body.append("      if (lane == 31) sg_tot = v_;")
        body.append("      sg_cnt[lane] = 0;")
        if cfg.cmajor == 3:
            body.append("      if (lane == 0) sg_next = 0;")
        body.append("    }")
        body.append("    __syncthreads();")
        psi_of = (lambda sub: str(t.psi[0])) if (t.K == 1 or t.uniform_psi) else (lambda sub: f"sg_psi[{sub}]")
        if t.K == 1:
            psi_of = lambda sub: "0"   # noqa: E731
        body.append(f"    for (int i_ = threadIdx.x; i_ < {M * TQ}; i_ += {Bk}) {{")
        body.append("      const int k_ = sg_key[i_];")
        body.append("      if (k_ >= 0) { const int sb_ = k_ >> 16; "
                    f"sg_ord[sg_start[{psi_of('sb_')}] + (k_ & 0xffff)] = i_ | (sb_ << 16); }}")
        body.append("    }")
        body.append("    __syncthreads();")
        # phase 2: evaluate the pairs in psi order
        body.append("    const int tot = sg_tot;")
        pf = cfg.prefetch and fetch_mode in ("table", "uniform")
        sctx["prefetched"] = bool(pf)
        dual = cfg.tpairs == 2
        cmajor = bool(cfg.cmajor) and not dual and not pf and t.K > 1
        if dual and not (cfg.coeffs == "table" and cfg.tloop and fetch_mode == "table"
                         and not smem_fetch and same_geom):
            raise ValueError("tpairs=2 needs coeffs='table', tloop=1 and per-sub-region offset tables")
        if pf:
            # software pipeline: pair pos + B's record, sub-region and coefficient gathers are
            # issued before pair pos's polynomial, so the gathers' latency hides behind it
            npad = t.n + 1 if t.n % 2 == 0 else t.n
            sten = t.stencils[0]
            st0 = strides[0]

            def pf_load(pre, posv):
                body.append(f"{pre}{{ const int e_ = sg_ord[{posv}];")
                body.append(f"{pre}  nf_pi = e_ & 0xffff; nf_sub = e_ >> 16;")
                body.append(f"{pre}  const float4 r_ = sg_rec[nf_pi];")
                for d in range(s):
                    body.append(f"{pre}  nf_u{d} = r_.{'xyz'[d]};")
                body.append(f"{pre}  const int b_ = __float_as_int(r_.w);")
                for j in range(t.n):
                    if fetch_mode == "table":
                        off = f"b_ + sg_off0[nf_sub * {npad} + {j}]"
                    else:
                        o = sum(sten[j][d] * st0[d] for d in range(s))
                        off = f"b_ + ({o})"
                    body.append(f"{pre}  nf_c{j} = __ldg((const float*)vol.base[0] + ({off}));")
                body.append(f"{pre}}}")
            body.append("    int nf_pi = 0, nf_sub = 0;")
            body.append("    float " + ", ".join([f"nf_u{d} = 0.f" for d in range(s)]
                                                + [f"nf_c{j} = 0.f" for j in range(t.n)]) + ";")
            body.append("    if ((int)threadIdx.x < tot)")
            pf_load("      ", "threadIdx.x")
            body.append(f"    for (int pos = threadIdx.x; pos < tot; pos += {Bk}) {{")
            body.append("      const int pi_ = nf_pi;")
            body.append("      const int sub = nf_sub;")
            for d in range(s):
                body.append(f"      const float u{d} = nf_u{d};")
            for j in range(t.n):
                body.append(f"      const float pfc{j} = nf_c{j};")
            body.append(f"      if (pos + {Bk} < tot)")
            pf_load("        ", f"pos + {Bk}")
            body.append(f"      const float* __restrict__ V = (const float*)vol.base[0];")
            body.append("      const int base = 0;")
        elif dual:
            # two pairs per thread (adjacent in psi order: the same polynomial except at a
            # class boundary, which takes the one-pair path below)
            body.append(f"    for (int pos = 2 * (int)threadIdx.x; pos < tot; pos += {2 * Bk}) {{")
            body.append("      const bool hasB = pos + 1 < tot;")
            body.append("      const int eA = sg_ord[pos], eB = sg_ord[hasB ? pos + 1 : pos];")
            body.append("      const int piA = eA & 0xffff, subA = eA >> 16, piB = eB & 0xffff, subB = eB >> 16;")
            body.append(f"      const int psiA = {psi_of('subA')}, psiB = {psi_of('subB')};")
            body.append(f"      const float* __restrict__ V = (const float*)vol.base[0];")
            body.append("      if (hasB && psiA == psiB) {")
            body.append("        const float4 rA = sg_rec[piA], rB = sg_rec[piB];")
            for d in range(s):
                body.append(f"        const float uA{d} = rA.{'xyz'[d]}, uB{d} = rB.{'xyz'[d]};")
            body.append("        const int baseA = __float_as_int(rA.w), baseB = __float_as_int(rB.w);")
            body.append("        const int psi = psiA;")
            body.append("        const int sub = subA, base = baseA;")
            em.lines = []
            em.indent = "        "
            sctx["dual"] = True
            emit_coset(0, False, phase="eval")
            sctx["dual"] = False
            body.extend(em.lines)
            body.append("      } else {")
            body.append("      for (int h_ = 0; h_ < (hasB ? 2 : 1); ++h_) {")
            body.append("      const int pi_ = h_ ? piB : piA;")
            body.append("      const int sub = h_ ? subB : subA;")
            body.append("      const float4 rec = sg_rec[pi_];")
            for d in range(s):
                body.append(f"      const float u{d} = rec.{'xyz'[d]};")
            body.append("      const int base = __float_as_int(rec.w);")
        elif cfg.cmajor == 3 and cmajor:
            # warp-sized chunks of the psi-ordered pairs handed out in order (shared counter):
            # the chunks in flight are a contiguous window of the order, i.e. at most two
            # polynomials' code is live in the SM, with no barrier between polynomials
            body.append("    for (;;) {")
            body.append("      int ch_ = 0;")
            body.append("      if (lane == 0) ch_ = atomicAdd(&sg_next, 1);")
            body.append("      ch_ = __shfl_sync(0xffffffffu, ch_, 0);")
            body.append("      if (ch_ * 32 >= tot) break;")
            if cfg.cflip and not render:
                # odd tiles walk the psi order backwards (chunks stay contiguous runs)
                body.append("      const int r_ = ch_ * 32 + (int)lane;")
                body.append("      if (r_ >= tot) continue;")
                body.append("      const int pos = sg_par ? tot - 1 - r_ : r_;")
            else:
                body.append("      const int pos = ch_ * 32 + (int)lane;")
                body.append("      if (pos >= tot) continue;")
            body.append("      const int e_ = sg_ord[pos];")
            body.append("      const int pi_ = e_ & 0xffff;")
            body.append("      const int sub = e_ >> 16;")
            body.append("      const float4 rec = sg_rec[pi_];")
            for d in range(s):
                body.append(f"      const float u{d} = rec.{'xyz'[d]};")
            body.append("      const int base = __float_as_int(rec.w);")
            body.append(f"      const float* __restrict__ V = (const float*)vol.base[0];")
        elif cmajor:
            # class-major: one reference polynomial at a time for the whole CTA (its code
            # stays in the SM's instruction cache); thread t keeps the positions p = t mod B
            # of the unsorted loop, so the work per thread is unchanged
            body.append(f"    for (int cls = 0; cls < {t.K}; ++cls) {{")
            body.append("      const int c0 = sg_start[cls];")
            body.append(f"      const int c1 = cls + 1 < {min(t.K, 32)} ? sg_start[cls + 1] : tot;")
            body.append(f"      for (int pos = c0 + ((((int)threadIdx.x - c0) % {Bk}) + {Bk}) % {Bk}; pos < c1; pos += {Bk}) {{")
            body.append("      const int e_ = sg_ord[pos];")
            body.append("      const int pi_ = e_ & 0xffff;")
            body.append("      const int sub = e_ >> 16;")
            body.append("      const float4 rec = sg_rec[pi_];")
            for d in range(s):
                body.append(f"      const float u{d} = rec.{'xyz'[d]};")
            body.append("      const int base = __float_as_int(rec.w);")
            body.append(f"      const float* __restrict__ V = (const float*)vol.base[0];")
        else:
            body.append(f"    for (int pos = threadIdx.x; pos < tot; pos += {Bk}) {{")
            body.append("      const int e_ = sg_ord[pos];")
            body.append("      const int pi_ = e_ & 0xffff;")
            body.append("      const int sub = e_ >> 16;")
            body.append("      const float4 rec = sg_rec[pi_];")
            for d in range(s):
                body.append(f"      const float u{d} = rec.{'xyz'[d]};")
            body.append("      const int base = __float_as_int(rec.w);")
            body.append(f"      const float* __restrict__ V = (const float*)vol.base[0];")
        if t.K > 1:
            body.append(f"      const int psi = {'cls' if (cmajor and cfg.cmajor != 3) else psi_of('sub')};")
        body.append("      float acc = 0.0f;")
        if cfg.grad:
            for d in range(s):
                body.append(f"      float gacc{d} = 0.0f;")
        em.lines = []
        em.indent = "      "
        emit_coset(0, False, phase="eval")
        body.extend(em.lines)
        if cfg.grad:
            g = ", ".join([f"gacc{d}" for d in range(s)] + ["0.0f"] * (3 - s))
            body.append(f"      sg_res4[pi_] = make_float4(acc, {g});")
        else:
            body.append("      sg_res[pi_] = acc;")
        if dual:
            body.append("      }")   # one-pair loop
            body.append("      }")   # one-pair path
        if cmajor and cfg.cmajor != 3:
            body.append("      }")   # positions of this class
            if cfg.cmajor == 2:
                body.append("      __syncthreads();")
        body.append("    }")
        body.append("    __syncthreads();")
        if render:
            # phase 3 (render): each of the RB first threads composites its ray's SJ samples
            # front to back (coset contributions summed in coset order)
            body.append(f"    if (threadIdx.x < {RB}) {{")
            body.append(f"      for (int jj = 0; jj < {TQ // RB} && j0 + jj < steps; ++jj) {{")
            body.append(f"        const int ql = jj * {RB} + (int)threadIdx.x;")
            if cfg.grad:
                body.append("        float4 a_ = sg_res4[ql];")
                for l in range(1, M):
                    body.append(f"        {{ const float4 b_ = sg_res4[{l * TQ} + ql]; a_.x += b_.x; a_.y += b_.y; a_.z += b_.z; a_.w += b_.w; }}")
                body.append("        const float acc = a_.x, gacc0 = a_.y, gacc1 = a_.z, gacc2 = a_.w;")
            else:
                expr = "sg_res[ql]"
                for l in range(1, M):
                    expr = f"({expr} + sg_res[{l * TQ} + ql])"
                body.append(f"        const float acc = 0.0f + {expr};")
            body.append("        const float dn = fminf(fmaxf((acc - tf_lo) * tf_inv, 0.f), 1.f);")
            body.append("        const float al = fminf(dn * my_aop, 1.f);")
            if cfg.grad:
                body.append("        const float gl = sqrtf(gacc0 * gacc0 + gacc1 * gacc1 + gacc2 * gacc2);")
                body.append("        const float sh = gl > 0.f ? 0.3f + 0.7f * fabsf(gacc0 * L0 + gacc1 * L1 + gacc2 * L2) / gl : 1.f;")
            else:
                body.append("        const float sh = 1.f;")
            body.append("        const float w = (1.f - A) * al * sh;")
            body.append("        C0 += w * (c0lo + dn * c0d);")
            body.append("        C1 += w * (c1lo + dn * c1d);")
            body.append("        C2 += w * (c2lo + dn * c2d);")
            body.append("        A += (1.f - A) * al;")
            body.append("      }")
            body.append("    }")
            body.append("    __syncthreads();")
            body.append("  }")   # step chunks
            body.append(f"  if (threadIdx.x < {RB} && myray < n) {stf}(&rgba[myray], make_float4(C0, C1, C2, A));")
            body.append("  __syncthreads();   // sg_rb0 is rewritten by the next claim")
            body.append("  }")   # ray blocks
            body.append("}")
    if sorted_ and not render:
        # phase 3: coset contributions summed in coset order, coalesced stores
        body.append(f"    for (int ql = threadIdx.x; ql < {TQ}; ql += {Bk}) {{")
        if presort:
            body.append("      if (q0 + ql >= n) break;")
            body.append("      const long long qi = (long long)sg_qidx[ql];")
        else:
            body.append("      const long long qi = q0 + ql;")
            body.append("      if (qi >= n) break;")
        if cfg.grad:
            body.append("      float4 a_ = sg_res4[ql];")
            for l in range(1, M):
                body.append(f"      {{ const float4 b_ = sg_res4[{l * TQ} + ql]; a_.x += b_.x; a_.y += b_.y; a_.z += b_.z; a_.w += b_.w; }}")
            body.append(f"      {stf}(&out[qi], a_.x);")
            for d in range(s):
                body.append(f"      {stf}(&grad[qi * {s} + {d}], a_.{'yzw'[d]});")
        else:
            expr = "sg_res[ql]"
            for l in range(1, M):
                expr = f"({expr} + sg_res[{l * TQ} + ql])"
            body.append(f"      {stf}(&out[qi], 0.0f + {expr});")
        body.append("    }")
        body.append("    __syncthreads();")
        body.append("  }")   # tile loop
        body.append("}")
    elif sorted_:
        pass
    elif pack2:
        emit_pack2_body()
    elif M == 1:
        em.line("{")
        em.indent = "    "
        emit_coset(0, False)
        em.indent = "  "
        em.line("}")
    elif cfg.unroll_cosets:
        for l in range(M):
            em.line(f"{{  // coset {l}")
            em.indent = "    "
            emit_coset(l, False)
            em.indent = "  "
            em.line("}")
    else:
        em.line("#pragma unroll 1")
        em.line(f"for (int l = 0; l < {M}; ++l) {{")
        em.indent = "    "
        emit_coset(None, True)
        em.indent = "  "
        em.line("}")
    if render and not sorted_:
        body += em.lines
        body.append("  const float dn = fminf(fmaxf((acc - tf_lo) * tf_inv, 0.f), 1.f);")
        body.append("  const float al = fminf(dn * aop, 1.f);")
        if cfg.grad:
            body.append("  const float gl = sqrtf(gacc0 * gacc0 + gacc1 * gacc1 + gacc2 * gacc2);")
            body.append("  const float sh = gl > 0.f ? 0.3f + 0.7f * fabsf(gacc0 * L0 + gacc1 * L1 + gacc2 * L2) / gl : 1.f;")
        else:
            body.append("  const float sh = 1.f;")
        body.append("  const float w = (1.f - A) * al * sh;")
        body.append("  C0 += w * (c0lo + dn * c0d);")
        body.append("  C1 += w * (c1lo + dn * c1d);")
        body.append("  C2 += w * (c2lo + dn * c2d);")
        body.append("  A += (1.f - A) * al;")
        body.append("  }")   # sample loop
        body.append(f"  {stf}(&rgba[qi], make_float4(C0, C1, C2, A));")
        body.append("  }")   # ray loop
        body.append("}")
    elif pack2:
        pass
    elif not sorted_:
        body += em.lines
        body.append(f"  {stf}(&out[qi], acc);")
        if cfg.grad:
            for d in range(s):
                body.append(f"  {stf}(&grad[qi * {s} + {d}], gacc{d});")
        body.append("  }")   # query loop (grid-stride in direct mode, chunk loop in binned mode)
        body.append("}")
    if lut:
        lit = ", ".join(flit(Fraction(v), fw) for v in lut)
        head.append(f"__constant__ {T} sg_lut[{len(lut)}] = {{{lit}}};")
    src = "\n".join(head + body) + "\n"
    return CudaProgram(
        name=space.name, source=src, entry=ENTRY, dim=s, ncosets=M, float_width=fw,
        block=cfg.block, halo=H, extents=ext, padded_extents=pext, has_grad=cfg.grad,
        has_dbg=cfg.dbg, config=cfg, space=space,
        mode=cfg.mode, bin=bin_ if binned else 0, brick=tuple(brick) if binned else (),
        smem_bytes=smem_bytes if binned else (sorted_smem if sorted_ else 0),
        stage_tma=binned and cfg.stage == "tma",
        chunk=cfg.chunk if binned else 0,
        queries_per_thread=cfg.tile // cfg.block if sorted_ else 1,
        presort=presort,
        rounding=(0 if (rm0.shape == PARALLELEPIPED and rm0.rounding == "floor") else 1),
        meta={"fetch_mode": fetch_mode, "K": t.K, "nsub": t.nsub, "n": t.n, "reach": h,
              "smem_tables": [x[0] for x in smem], "lut_entries": len(lut)})
