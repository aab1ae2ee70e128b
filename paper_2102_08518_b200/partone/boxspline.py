"""Exact (rational) box-spline evaluation.

M_Xi(x) for a multiset Xi of n direction vectors spanning R^s is evaluated with
the de Boor-Hoellig recurrence

    (n - s) M_Xi(x) = sum_{xi in Xi} [ t_xi M_{Xi\\xi}(x) + (1 - t_xi) M_{Xi\\xi}(x - xi) ],
    for any t with Xi t = x,

down to s directions, where M_B = 1/|det B| on the half-open parallelepiped
B [0,1)^s.  Terms whose remaining multiset no longer spans R^s are zero
almost everywhere.  Points are expected off the knot planes (the producer only
samples interiors of the arrangement's regions), so the half-open convention
never decides a value.  Everything is `Fraction`, memoized on
(multiplicity vector, x).

A spline basis function is a weighted sum of shifted box splines
(`BoxSum`): a single centered box spline for the box-spline spaces, and the
zonotope-tiling expansion of the Voronoi cell's indicator convolved k times
for the Voronoi splines (voronoi.py).
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field
from fractions import Fraction
from functools import lru_cache

from .. import exact


def _vec(v):
    return tuple(Fraction(x) for x in v)


def _rank(vectors, s):
    rows = [list(v) for v in vectors]
    r = 0
    for c in range(s):
        p = next((i for i in range(r, len(rows)) if rows[i][c] != 0), None)
        if p is None:
            continue
        rows[r], rows[p] = rows[p], rows[r]
        for i in range(len(rows)):
            if i != r and rows[i][c] != 0:
                f = rows[i][c] / rows[r][c]
                rows[i] = [a - f * b for a, b in zip(rows[i], rows[r])]
        r += 1
    return r


class BoxSpline:
    """M_Xi with distinct directions `dirs` and multiplicities `mult`."""

    def __init__(self, dirs, mult=None):
        dirs = [_vec(d) for d in dirs]
        self.s = len(dirs[0])
        # merge parallel-equal duplicates
        merged = {}
        for i, d in enumerate(dirs):
            m = 1 if mult is None else int(mult[i])
            merged[d] = merged.get(d, 0) + m
        self.dirs = tuple(merged)
        self.mult = tuple(merged[d] for d in self.dirs)
        if _rank(self.dirs, self.s) < self.s:
            raise ValueError("directions do not span R^s")
        self._cache = {}

    @property
    def n(self):
        return sum(self.mult)

    @property
    def degree(self):
        return self.n - self.s

    def support_box(self):
        """Axis-aligned bounds of the zonotope sum_i [0, xi_i]."""
        lo = [Fraction(0)] * self.s
        hi = [Fraction(0)] * self.s
        for d, m in zip(self.dirs, self.mult):
            for a in range(self.s):
                if d[a] < 0:
                    lo[a] += m * d[a]
                else:
                    hi[a] += m * d[a]
        return lo, hi

    def center(self):
        return tuple(sum(m * d[a] for d, m in zip(self.dirs, self.mult)) / 2 for a in range(self.s))

    def __call__(self, x):
        return self._eval(self.mult, _vec(x))

    def _spans(self, mult):
        return _rank([d for d, m in zip(self.dirs, mult) if m], self.s) == self.s

    def _eval(self, mult, x):
        key = (mult, x)
        c = self._cache.get(key)
        if c is not None:
            return c
        s = self.s
        n = sum(mult)
        if n == s:
            vecs = [d for d, m in zip(self.dirs, mult) for _ in range(m)]
            if _rank(vecs, s) < s:
                val = Fraction(0)
            else:
                B = tuple(tuple(vecs[j][i] for j in range(s)) for i in range(s))  # columns
                t = exact.matvec(exact.inverse(B), x)
                inside = all(0 <= v < 1 for v in t)
                val = Fraction(1) / abs(exact.det(B)) if inside else Fraction(0)
            self._cache[key] = val
            return val
        # quick support rejection
        lo = [Fraction(0)] * s
        hi = [Fraction(0)] * s
        for d, m in zip(self.dirs, mult):
            for a in range(s):
                if d[a] < 0:
                    lo[a] += m * d[a]
                else:
                    hi[a] += m * d[a]
        if any(x[a] <= lo[a] or x[a] >= hi[a] for a in range(s)):
            self._cache[key] = Fraction(0)
            return Fraction(0)
        # t supported on a basis subset: t_B = B^{-1} x
        basis = []
        for i, (d, m) in enumerate(zip(self.dirs, mult)):
            if m and _rank([self.dirs[j] for j in basis] + [d], s) == len(basis) + 1:
                basis.append(i)
            if len(basis) == s:
                break
        B = tuple(tuple(self.dirs[j][a] for j in basis) for a in range(s))
        tb = exact.matvec(exact.inverse(B), x)
        tval = {j: tb[k] for k, j in enumerate(basis)}
        total = Fraction(0)
        for i, (d, m) in enumerate(zip(self.dirs, mult)):
            if not m:
                continue
            rest = mult[:i] + (m - 1,) + mult[i + 1:]
            if not self._spans(rest):
                continue
            ti = tval.get(i, Fraction(0))
            # the m copies of direction i: one carries t_i (if i in basis), the rest t = 0
            part = Fraction(0)
            a = self._eval(rest, x)
            b = self._eval(rest, tuple(xv - dv for xv, dv in zip(x, d)))
            # copy with t_i:
            part += ti * a + (1 - ti) * b
            # other copies (t = 0):
            part += (m - 1) * b
            total += part
        val = total / (n - s)
        self._cache[key] = val
        return val


@dataclass
class BoxTerm:
    weight: Fraction
    box: BoxSpline
    shift: tuple     # phi contribution: weight * M(x - shift)


@dataclass
class BoxSum:
    """phi(x) = sum_t w_t M_{Xi_t}(x - s_t)."""
    s: int
    terms: list = field(default_factory=list)

    def __call__(self, x):
        x = _vec(x)
        total = Fraction(0)
        for t in self.terms:
            total += t.weight * t.box(tuple(a - b for a, b in zip(x, t.shift)))
        return total

    def degree(self):
        return max(t.box.degree for t in self.terms)

    def support_box(self):
        lo = [None] * self.s
        hi = [None] * self.s
        for t in self.terms:
            l, h = t.box.support_box()
            for a in range(self.s):
                la, ha = l[a] + t.shift[a], h[a] + t.shift[a]
                lo[a] = la if lo[a] is None else min(lo[a], la)
                hi[a] = ha if hi[a] is None else max(hi[a], ha)
        return lo, hi

    def knot_planes(self):
        """{(primitive integer normal a, offset o)}: planes a.x = o of every term."""
        out = set()
        for t in self.terms:
            bx = t.box
            s = self.s
            for combo in itertools.combinations(range(len(bx.dirs)), s - 1):
                vecs = [bx.dirs[i] for i in combo]
                if _rank(vecs, s) < s - 1:
                    continue
                a = _normal(vecs, s)
                # knots pass through shift + subset sums of all directions (with multiplicity)
                offs = {Fraction(0)}
                for d, m in zip(bx.dirs, bx.mult):
                    ad = sum(x * y for x, y in zip(a, d))
                    offs = {o + k * ad for o in offs for k in range(m + 1)}
                base = sum(x * y for x, y in zip(a, t.shift))
                for o in offs:
                    out.add((a, base + o))
        return out


def _normal(vecs, s):
    """Primitive integer normal to the span of s-1 vectors, lexicographically positive."""
    if s == 1:
        n = [Fraction(1)]
    else:
        # generalized cross product via cofactors
        M = [list(v) for v in vecs]
        n = []
        for i in range(s):
            minor = tuple(tuple(row[j] for j in range(s) if j != i) for row in M)
            n.append(((-1) ** i) * exact.det(minor) if minor else Fraction(1))
    return primitive(n)


def primitive(v):
    from math import gcd
    den = 1
    for q in v:
        den = den * Fraction(q).denominator // gcd(den, Fraction(q).denominator)
    ints = [int(Fraction(q) * den) for q in v]
    g = 0
    for x in ints:
        g = gcd(g, abs(x))
    ints = [x // g for x in ints]
    for x in ints:
        if x != 0:
            if x < 0:
                ints = [-y for y in ints]
            break
    return tuple(Fraction(x) for x in ints)


def centered_box(dirs, mult=None) -> BoxSum:
    """phi(x) = M_Xi(x + center): the box spline centered at the origin."""
    bx = BoxSpline(dirs, mult)
    c = bx.center()
    return BoxSum(bx.s, [BoxTerm(Fraction(1), bx, tuple(-v for v in c))])
