"""Symbolic polynomial pieces of box splines (exact).

The de Boor-Hoellig recurrence used for point values in boxspline.py holds
identically in x on every region of the knot-plane arrangement, with
t(x) = B^{-1} x linear in x.  Running it on polynomials instead of numbers
gives the polynomial piece of M_Xi on the region containing a generic point
p directly:

    (n - s) P_Xi,p(x) = sum_xi [ t_xi(x) P_{Xi\\xi},p(x)
                                 + (1 - t_xi(x)) P_{Xi\\xi},p-xi(x - xi) ]

down to s directions, where the piece of 1/|det B| chi_{B[0,1)^s} is a constant.
One recursive call replaces the C(deg+s, s) point evaluations plus the
Vandermonde solve of an interpolation fit; the producer still certifies every
piece against independent point values of boxspline.BoxSpline.

Polynomials are dicts {exponent tuple: Fraction}; memoization is global over
(direction multiset, point) so the many box-spline terms of a Voronoi spline
share their sub-problems.
"""

from __future__ import annotations

from fractions import Fraction
from math import comb

from .. import exact
from .boxspline import BoxSum, _rank

F = Fraction


def padd(a, b, scale=1):
    out = dict(a)
    for e, c in b.items():
        v = out.get(e, F(0)) + scale * c
        if v:
            out[e] = v
        else:
            out.pop(e, None)
    return out


def pscale(a, k):
    if k == 0:
        return {}
    return {e: c * k for e, c in a.items()}


def pmul_linear(a, lin, const):
    """a(x) * (lin . x + const)."""
    out = {}
    s = len(lin)
    for e, c in a.items():
        if const:
            out[e] = out.get(e, F(0)) + c * const
        for d in range(s):
            if lin[d]:
                e2 = e[:d] + (e[d] + 1,) + e[d + 1:]
                out[e2] = out.get(e2, F(0)) + c * lin[d]
    return {e: c for e, c in out.items() if c}


def pshift(a, v):
    """a(x - v)."""
    if not any(v):
        return dict(a)
    out = {}
    s = len(v)
    for e, c in a.items():
        # expand prod_d (x_d - v_d)^{e_d}
        terms = [((), c)]
        for d in range(s):
            nxt = []
            for k in range(e[d] + 1):
                f = comb(e[d], k) * (-v[d]) ** (e[d] - k)
                if f == 0:
                    continue
                for ex, cc in terms:
                    nxt.append((ex + (k,), cc * f))
            terms = nxt
        for ex, cc in terms:
            out[ex] = out.get(ex, F(0)) + cc
    return {e: c for e, c in out.items() if c}


def peval(a, x):
    tot = F(0)
    for e, c in a.items():
        t = c
        for xi, ei in zip(x, e):
            if ei:
                t *= xi ** ei
        tot += t
    return tot


class PieceEvaluator:
    def __init__(self, s):
        self.s = s
        self._memo = {}
        self._basis = {}

    def piece(self, dirs, mult, p):
        """Polynomial of M_{dirs^mult} on the region containing generic point p."""
        key = (dirs, mult, p)
        r = self._memo.get(key)
        if r is not None:
            return r
        r = self._piece(dirs, mult, p)
        self._memo[key] = r
        return r

    def _spans(self, dirs, mult):
        return _rank([d for d, m in zip(dirs, mult) if m], self.s) == self.s

    def _piece(self, dirs, mult, p):
        s = self.s
        n = sum(mult)
        zero = (0,) * s
        # support box rejection
        for a in range(s):
            lo = sum(m * d[a] for d, m in zip(dirs, mult) if d[a] < 0)
            hi = sum(m * d[a] for d, m in zip(dirs, mult) if d[a] > 0)
            if p[a] <= lo or p[a] >= hi:
                return {}
        if n == s:
            vecs = [d for d, m in zip(dirs, mult) for _ in range(m)]
            if _rank(vecs, s) < s:
                return {}
            B = tuple(tuple(vecs[j][i] for j in range(s)) for i in range(s))
            t = exact.matvec(exact.inverse(B), p)
            if all(0 < v < 1 for v in t):
                return {zero: F(1) / abs(exact.det(B))}
            return {}
        bkey = (dirs, mult)
        bas = self._basis.get(bkey)
        if bas is None:
            basis = []
            for i, (d, m) in enumerate(zip(dirs, mult)):
                if m and _rank([dirs[j] for j in basis] + [d], s) == len(basis) + 1:
                    basis.append(i)
                if len(basis) == s:
                    break
            B = tuple(tuple(dirs[j][a] for j in basis) for a in range(s))
            Binv = exact.inverse(B)
            bas = (basis, {j: Binv[k] for k, j in enumerate(basis)})
            self._basis[bkey] = bas
        basis, rows = bas
        total = {}
        for i, (d, m) in enumerate(zip(dirs, mult)):
            if not m:
                continue
            rest = mult[:i] + (m - 1,) + mult[i + 1:]
            if not self._spans(dirs, rest):
                continue
            pb = tuple(pv - dv for pv, dv in zip(p, d))
            b = pshift(self.piece(dirs, rest, pb), d)       # M_rest(x - xi) near p
            if i in rows:
                a = self.piece(dirs, rest, p)
                lin = rows[i]                                # t_i(x) = row . x
                total = padd(total, pmul_linear(a, lin, F(0)))
                total = padd(total, b)
                total = padd(total, pmul_linear(b, lin, F(0)), -1)
                if m > 1:
                    total = padd(total, pscale(b, m - 1))
            else:
                total = padd(total, pscale(b, m))
        return pscale(total, F(1, n - s))


def phi_piece(phi: BoxSum, ev: PieceEvaluator, p, site=None):
    """Polynomial (in x) of phi(x - site) on the region containing generic point p."""
    s = phi.s
    site = tuple(F(v) for v in (site or (0,) * s))
    out = {}
    for t in phi.terms:
        shift = tuple(a + b for a, b in zip(site, t.shift))
        q = tuple(a - b for a, b in zip(p, shift))
        pc = ev.piece(t.box.dirs, t.box.mult, q)
        if pc:
            out = padd(out, pscale(pshift(pc, shift), t.weight))
    return out
