"""CPU oracle for the spline-reconstruction hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain numpy restatement of the reference evaluator
`splinegen.oracle.reference_eval_batch` (reference: pkg/src/splinegen/oracle.py:77-104)
and of the pieces it calls.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it, and only
as the checker or the timed CPU baseline -- never as a product code path.

It is deliberately self-contained: it has its own reader for the JSON space
format (reference schema: pkg/README.md "Description file format",
pkg/src/splinegen/model.py:205-300) so that it shares no code with the
product package it checks.

Pinning: `tests/golden/make_golden.py` runs the *actual* reference package
(imported from /root/reference in the build container) on seeded inputs and
commits its outputs under tests/golden/; `tests/test_oracle_golden.py` checks
this restatement against those vectors bit-for-bit (values, lattice shifts k
and sub-region indices).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

NO_SYMBOL = -1
UNREACHABLE = -1


class UnreachableRegionError(Exception):
    """Mirrors splinegen.oracle.UnreachableRegionError (oracle.py:26)."""


# -- minimal exact reader for the space schema ---------------------------------


@dataclass(frozen=True)
class OSub:
    transform: tuple          # s x s Fractions
    shift: tuple              # s Fractions
    stencil: tuple            # n x s ints
    psi_index: int


@dataclass(frozen=True)
class OSpace:
    name: str
    dim: int
    cosets: tuple             # M x s Fractions
    generator: tuple
    shape: str                # "parallelepiped" | "voronoi"
    rounding: str             # "floor" | "round_nearest"
    basis: tuple | None
    planes: tuple             # ((normal Fractions), offset Fraction)
    modulus: int
    sigma: tuple
    subregions: tuple
    ref_polys: tuple          # each: tuple of ((exps), c_index, Fraction) sorted

    @property
    def ncosets(self):
        return len(self.cosets)

    @property
    def stencil_size(self):
        return len(self.subregions[0].stencil)


def _q(v) -> Fraction:
    if isinstance(v, bool) or isinstance(v, float):
        raise ValueError("non-exact literal")
    return Fraction(v)


def load_space(text: str) -> OSpace:
    """Parse the JSON description (no validation; reference model.py:226-300)."""
    doc = json.loads(text)
    dim = int(doc["dim"])
    lat = doc["lattice"]
    rm = doc["region_map"]
    basis = None
    if rm.get("basis") is not None:
        basis = tuple(tuple(_q(v) for v in row) for row in rm["basis"])
    planes = tuple(
        (tuple(_q(v) for v in p["normal"]), _q(p["offset"])) for p in doc["planes"]
    )
    subs = tuple(
        OSub(
            transform=tuple(tuple(_q(v) for v in row) for row in s["transform"]),
            shift=tuple(_q(v) for v in s["shift"]),
            stencil=tuple(tuple(int(v) for v in site) for site in s["stencil"]),
            psi_index=int(s["psi_index"]),
        )
        for s in doc["subregions"]
    )
    polys = []
    for monos in doc["ref_polys"]:
        terms = {}
        for m in monos:
            key = (tuple(int(e) for e in m["x_exps"]), int(m["c_index"]))
            terms[key] = terms.get(key, Fraction(0)) + _q(m["coeff"])
        # Poly.sorted_terms order: key (exps, c_index) ascending (poly.py:26-27, 70-73)
        polys.append(tuple((k[0], k[1], c) for k, c in sorted(terms.items()) if c != 0))
    return OSpace(
        name=doc.get("name", "unnamed"),
        dim=dim,
        cosets=tuple(tuple(_q(v) for v in c) for c in lat["cosets"]),
        generator=tuple(tuple(_q(v) for v in row) for row in lat["generator"]),
        shape=rm["shape"],
        rounding=rm["rounding"],
        basis=basis,
        planes=planes,
        modulus=int(doc["indexer"]["modulus"]),
        sigma=tuple(int(v) for v in doc["indexer"]["sigma"]),
        subregions=subs,
        ref_polys=tuple(polys),
    )


def load_space_file(path) -> OSpace:
    with open(path, "r", encoding="utf-8") as fh:
        return load_space(fh.read())


# -- exact helpers (reference exact.py) ----------------------------------------


def _is_identity(m) -> bool:
    return all(m[i][j] == (1 if i == j else 0) for i in range(len(m)) for j in range(len(m)))


def _mat_vec(m, v):
    return tuple(sum(row[j] * v[j] for j in range(len(v))) for row in m)


def _float_mat(m) -> np.ndarray:
    return np.array([[float(q) for q in row] for row in m])


# -- the evaluation recipe (reference oracle.py:34-104) ------------------------


def round_half_away(v: np.ndarray) -> np.ndarray:
    """oracle.py:34-35: floor(v+0.5) for v >= 0, ceil(v-0.5) otherwise (f64)."""
    return np.where(v >= 0, np.floor(v + 0.5), np.ceil(v - 0.5))


def rho(space: OSpace, xl: np.ndarray):
    """oracle.py:38-53: (integer shift k, local point xl - k)."""
    if space.shape == "parallelepiped":
        basis = _float_mat(space.basis)
        identity = _is_identity(space.basis)
        rounding = space.rounding
    else:
        basis = np.eye(space.dim)
        identity = True
        rounding = "round_nearest"
    u = xl if identity else xl @ np.linalg.inv(basis).T
    r = round_half_away(u) if rounding == "round_nearest" else np.floor(u)
    k = r if identity else r @ basis.T
    k = k.astype(np.int64)
    return k, xl - k.astype(xl.dtype)


def plane_q(space: OSpace, xs: np.ndarray) -> np.ndarray:
    """oracle.py:56-66 up to the modulus: q = sum_i [normal_i . x >= offset_i] << i."""
    n = xs.shape[0]
    q = np.zeros(n, dtype=np.int64)
    for i, (normal, offset) in enumerate(space.planes):
        nv = np.array([float(v) for v in normal])
        dot = xs @ nv
        q |= (dot >= float(offset)).astype(np.int64) << i
    return q % space.modulus


def membership(space: OSpace, xs: np.ndarray) -> np.ndarray:
    """oracle.py:56-74: sub-region index per point; sigma == -1 raises."""
    n = xs.shape[0]
    if not space.planes:
        return np.zeros(n, dtype=np.int64)
    q = plane_q(space, xs)
    sigma = np.array(space.sigma, dtype=np.int64)
    idx = sigma[q]
    if (idx == UNREACHABLE).any():
        bad = int(q[idx == UNREACHABLE][0])
        raise UnreachableRegionError(f"point classified into unreachable sigma entry q={bad}")
    return idx


def fetch(arr: np.ndarray, coords) -> np.ndarray:
    """ir.py:555-558: periodic C-order fetch, coords % extents."""
    idx = tuple(np.asarray(c) % e for c, e in zip(coords, arr.shape))
    return arr[idx]


def poly_eval(terms, x, c=()):
    """poly.py:135-150: sum of terms in sorted order, float64 semantics."""
    total = 0.0
    for exps, ci, coeff in terms:
        term = float(coeff)
        for k, e in enumerate(exps):
            if e:
                term = term * x[k] ** e
        if ci != NO_SYMBOL:
            term = term * c[ci]
        total = total + term
    return total


def diff_terms(terms, axis):
    """poly.py:169-179: exact partial derivative, re-sorted like Poly.sorted_terms."""
    out = {}
    for exps, ci, coeff in terms:
        e = exps[axis]
        if e == 0:
            continue
        new = tuple(v - 1 if k == axis else v for k, v in enumerate(exps))
        out[(new, ci)] = out.get((new, ci), Fraction(0)) + coeff * e
    return tuple((k[0], k[1], c) for k, c in sorted(out.items()) if c != 0)


def _tshift(sub: OSub):
    """codegen.py:126-134: t' = -T.t folded exactly."""
    return tuple(-v for v in _mat_vec(sub.transform, sub.shift))


def selection(space: OSpace, xs):
    """Per coset: (k (N,s) int64, sub-region index (N,) int64) -- oracle.py:85-89."""
    xs = np.asarray(xs, dtype=np.float64)
    out = []
    for offset in space.cosets:
        xl = xs - np.array([float(q) for q in offset])
        k, xloc = rho(space, xl)
        out.append((k, membership(space, xloc)))
    return out


def reference_eval_batch(space: OSpace, xs, arrays, grad: bool = False):
    """oracle.py:77-104 restated.  `arrays` is one C-order array per coset.

    With grad=True also returns the spatial gradient (N, s):
    sum over cosets of T^T . (d psi / d u) (restatement of the same recipe with
    psi.eval replaced by the exact derivative polynomials, poly.py:169-179).
    """
    xs = np.asarray(xs, dtype=np.float64)
    if xs.ndim != 2 or xs.shape[1] != space.dim:
        raise ValueError(f"expected points of shape (N, {space.dim})")
    if len(arrays) != space.ncosets:
        raise ValueError(f"data has {len(arrays)} cosets, space wants {space.ncosets}")
    n = xs.shape[0]
    s = space.dim
    total = np.zeros(n)
    gtotal = np.zeros((n, s)) if grad else None
    dpolys = None
    if grad:
        dpolys = [[diff_terms(p, a) for a in range(s)] for p in space.ref_polys]
    for ci, offset in enumerate(space.cosets):
        xl = xs - np.array([float(q) for q in offset])
        k, xloc = rho(space, xl)
        idx = membership(space, xloc)
        for j in np.unique(idx):
            sub = space.subregions[j]
            mask = idx == j
            t = _float_mat(sub.transform)
            tp = np.array([float(q) for q in _tshift(sub)])
            u = xloc[mask] @ t.T + tp
            km = k[mask]
            arr = np.asarray(arrays[ci])
            cvals = [fetch(arr, tuple(km[:, d] + site[d] for d in range(s))) for site in sub.stencil]
            uu = [u[:, d] for d in range(s)]
            total[mask] += poly_eval(space.ref_polys[sub.psi_index], uu, cvals)
            if grad:
                du = [poly_eval(dpolys[sub.psi_index][a], uu, cvals) * np.ones(int(mask.sum()))
                      for a in range(s)]
                for e in range(s):
                    acc = np.zeros(int(mask.sum()))
                    for a in range(s):
                        if t[a][e] != 0.0:
                            acc = acc + t[a][e] * du[a]
                    gtotal[mask, e] += acc
    if grad:
        return total, gtotal
    return total


# -- the convolution-sum oracle (reference oracle.py:115-177) -------------------


def support_radius(space: OSpace) -> float:
    reach = max(abs(int(v)) for sub in space.subregions for site in sub.stencil for v in site)
    if space.shape == "parallelepiped":
        roe = max(float(sum(abs(q) for q in row)) for row in space.basis)
        if space.rounding == "round_nearest":
            roe /= 2.0
    else:
        roe = 0.5
    return reach + roe


def delta_arrays(space: OSpace, radius: float | None = None):
    r = support_radius(space) if radius is None else radius
    extent = 2 * (int(math.ceil(r)) + 2) + 3
    shape = (extent,) * space.dim
    arrays = [np.zeros(shape) for _ in range(space.ncosets)]
    arrays[0][(0,) * space.dim] = 1.0
    return arrays


def basis_from_delta_batch(space: OSpace, ys, delta=None):
    if delta is None:
        delta = delta_arrays(space)
    return reference_eval_batch(space, ys, delta)


def convolution_eval_batch(space: OSpace, xs, arrays, radius: float | None = None):
    xs = np.asarray(xs, dtype=np.float64)
    r = support_radius(space) if radius is None else radius
    delta = delta_arrays(space, r)
    window = int(math.floor(r + 1.5))
    anchor = round_half_away(xs).astype(np.int64)
    total = np.zeros(xs.shape[0])
    offsets = np.stack(
        np.meshgrid(*([np.arange(-window, window + 1)] * space.dim), indexing="ij"), axis=-1
    ).reshape(-1, space.dim)
    for ci, coset in enumerate(space.cosets):
        shift = np.array([float(q) for q in coset])
        for w in offsets:
            z = anchor + w
            site = z.astype(np.float64) + shift
            values = fetch(np.asarray(arrays[ci]), tuple(z[:, d] for d in range(space.dim)))
            phi = basis_from_delta_batch(space, xs - site, delta)
            total += values * phi
    return total


# -- seeded inputs (reference bench.py:57-74) ----------------------------------


def make_volume(space: OSpace, extents, seed: int, float_width: str = "f64"):
    rng = np.random.default_rng(seed)
    dtype = np.float64 if float_width == "f64" else np.float32
    return [rng.random(tuple(int(e) for e in extents)).astype(dtype) for _ in range(space.ncosets)]


def sample_points(space: OSpace, arrays, count: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    spans = np.array(np.asarray(arrays[0]).shape, dtype=np.float64)
    return rng.random((count, space.dim)) * spans
