"""Stabilizer-symmetry reduction of a reference polynomial (kernel form "sym").

A reference polynomial psi(u, c) = sum_j c_j p_j(u) often has mirror symmetries
that survive the Part-I sub-region reduction: a flip u_a -> 2 z_a - u_a (z_a in
{0, 1/2}) that maps the stencil onto itself (site m -> m' with m'_a = 2 z_a - m_a)
and satisfies p_j(flip u) = p_{sigma(j)}(u) exactly.  For the abelian group F of
such flips, in the centred frame v = u - z every site orbit {g r : g in F}
contributes

    sum_g c_{g r} p_r(g v) = sum_e a_{r,e} v^e  s_{r, par(e)},
    s_{r,P} = sum_{g in F/Stab(r)} (-1)^{<P, g>} c_{g r}      (a Walsh-Hadamard mix)

so each orbit costs one polynomial's terms instead of |orbit| of them (the
tricubic B-spline drops from 1,728 terms to 8 x 64; the BCC quintic box spline's
reference region keeps one flip).  This is an exact algebraic rewrite of the
same polynomial; only the floating-point evaluation order changes.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass
from fractions import Fraction

from .poly import NO_SYMBOL, Poly


@dataclass
class SymForm:
    shift: tuple              # z: evaluate at v = u - z
    axes: tuple               # flip axes
    poly: Poly                # psi'(v, s) over the mixed symbols s
    mixes: list               # per new symbol: [(sign, site index j), ...]
    orbits: list              # (reps [(bits, j)], {parity bits P: symbol index})
    terms_before: int
    terms_after: int


def _flip_poly(p: Poly, a: int, z: Fraction) -> Poly:
    """p(u) with u_a -> 2 z - u_a."""
    s = p.dim
    A = [[Fraction(int(i == j)) for j in range(s)] for i in range(s)]
    A[a][a] = Fraction(-1)
    b = [Fraction(0)] * s
    b[a] = 2 * z
    return p.substitute_affine(A, b)


def find_flips(poly: Poly, stencil):
    """[(axis, z, sigma)] of exact mirror symmetries of (poly, stencil)."""
    s = poly.dim
    st = [tuple(m) for m in stencil]
    idx = {m: j for j, m in enumerate(st)}
    out = []
    for a in range(s):
        for z in (Fraction(0), Fraction(1, 2)):
            sigma = []
            ok = True
            for m in st:
                mm = tuple(int(2 * z - v) if k == a else v for k, v in enumerate(m))
                if mm not in idx:
                    ok = False
                    break
                sigma.append(idx[mm])
            if not ok:
                continue
            if all(_flip_poly(poly.coefficient_of(j), a, z) == poly.coefficient_of(sigma[j])
                   for j in range(len(st))):
                out.append((a, z, sigma))
                break
    return out


def symmetrize(poly: Poly, stencil) -> SymForm | None:
    flips = find_flips(poly, stencil)
    if not flips:
        return None
    s = poly.dim
    n = len(stencil)
    axes = tuple(a for a, _, _ in flips)
    shift = [Fraction(0)] * s
    for a, z, _ in flips:
        shift[a] = z
    # p_j in the centred frame v = u - z
    I = [[Fraction(int(i == j)) for j in range(s)] for i in range(s)]
    pj = [poly.coefficient_of(j).substitute_affine(I, shift) for j in range(n)]
    k = len(flips)
    perms = [f[2] for f in flips]

    def image(j, bits):
        for t in range(k):
            if bits >> t & 1:
                j = perms[t][j]
        return j

    seen = set()
    terms = {}
    mixes = []
    sym_of = {}
    orbits = []
    for r in range(n):
        if r in seen:
            continue
        reps = []
        imgs = set()
        for bits in range(1 << k):
            jj = image(r, bits)
            if jj not in imgs:
                imgs.add(jj)
                reps.append((bits, jj))
        seen |= imgs
        orbit_syms = {}
        orbits.append((reps, orbit_syms))
        for (e, _c), q in pj[r].terms.items():
            P = tuple(e[a] % 2 for a in axes)
            key = (r, P)
            if key not in sym_of:
                sym_of[key] = len(mixes)
                mix = []
                for bits, jj in reps:
                    par = sum(P[t] for t in range(k) if bits >> t & 1) % 2
                    mix.append((-1 if par else 1, jj))
                mixes.append(mix)
                orbit_syms[sum(P[t] << t for t in range(k))] = sym_of[key]
            tk = (e, sym_of[key])
            terms[tk] = terms.get(tk, Fraction(0)) + q
    free = {(e, NO_SYMBOL): q for (e, c), q in poly.terms.items() if c == NO_SYMBOL}
    if free:
        fp = Poly(s, free).substitute_affine(I, shift)
        for key, q in fp.terms.items():
            terms[key] = terms.get(key, Fraction(0)) + q
    newp = Poly(s, terms)
    return SymForm(shift=tuple(shift), axes=axes, poly=newp, mixes=mixes, orbits=orbits,
                   terms_before=len(poly.terms), terms_after=len(newp.terms))


def check(form: SymForm, poly: Poly, stencil, trials=4, seed=0) -> bool:
    """Exact equality of psi and psi' at random rational points / data."""
    import random
    rng = random.Random(seed)
    s = poly.dim
    for _ in range(trials):
        u = [Fraction(rng.randint(-500, 500), 997) for _ in range(s)]
        c = [Fraction(rng.randint(-500, 500), 991) for _ in range(len(stencil))]
        v = [a - b for a, b in zip(u, form.shift)]
        sv = [sum(sign * c[j] for sign, j in mix) for mix in form.mixes]
        if poly.eval_exact(u, c) != form.poly.eval_exact(v, sv):
            return False
    return True
