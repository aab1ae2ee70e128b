"""Voronoi splines as sums of shifted box splines.

The Voronoi cell V of the BCC lattice (truncated octahedron) and of the FCC
lattice (rhombic dodecahedron) are zonotopes Z(G) = sum_i [0, g_i].  A fine
zonotopal tiling (lower faces of a generic lifting) writes
    chi_Z = sum_{B basis of G} chi_{B [0,1)^s + z_B},
and chi_{B[0,1)^s} = |det B| M_B, so the order-k Voronoi spline
    V_k = chi_V * ... * chi_V  (k factors, centred)
is a weighted sum of box splines M_{B_1 u ... u B_k}(x + k c - sum z_{B_i}).
The producer normalizes to a partition of unity.  "Order k" follows the
paper's usage (order-2 Voronoi ~ tensor-product linear);
pieces have total degree (k - 1) * s.
"""

from __future__ import annotations

import itertools
import random
from fractions import Fraction

from .. import exact
from .boxspline import BoxSpline, BoxSum, BoxTerm, _rank

F = Fraction


def zonotope_tiles(gens, seed=7):
    """[(basis index triple, translation z_B)] of a fine zonotopal tiling of Z(gens)."""
    gens = [tuple(F(v) for v in g) for g in gens]
    s = len(gens[0])
    rng = random.Random(seed)
    heights = [F(rng.randint(1, 10 ** 6), 997) for _ in gens]
    lifted = [g + (h,) for g, h in zip(gens, heights)]
    tiles = []
    for combo in itertools.combinations(range(len(gens)), s):
        if _rank([gens[i] for i in combo], s) < s:
            continue
        # normal nu in R^{s+1} to the lifted basis, nu_{s} > 0
        rows = [lifted[i] for i in combo]
        nu = []
        for j in range(s + 1):
            minor = tuple(tuple(r[k] for k in range(s + 1) if k != j) for r in rows)
            nu.append(((-1) ** j) * exact.det(minor))
        if nu[s] < 0:
            nu = [-v for v in nu]
        z = [F(0)] * s
        for i in range(len(gens)):
            if i in combo:
                continue
            dot = sum(a * b for a, b in zip(nu, lifted[i]))
            if dot == 0:
                raise RuntimeError("non-generic lifting")
            if dot < 0:
                z = [a + b for a, b in zip(z, gens[i])]
        tiles.append((combo, tuple(z)))
    return tiles


def voronoi_spline(gens, order: int) -> BoxSum:
    """Order-k Voronoi spline (un-normalized) of the zonotope Z(gens), centred at 0."""
    gens = [tuple(F(v) for v in g) for g in gens]
    s = len(gens[0])
    center = tuple(sum(g[d] for g in gens) / 2 for d in range(s))
    tiles = zonotope_tiles(gens)
    dets = {}
    for combo, _ in tiles:
        B = tuple(tuple(gens[j][a] for j in combo) for a in range(s))
        dets[combo] = abs(exact.det(B))
    acc = {}
    for tup in itertools.product(range(len(tiles)), repeat=order):
        mult = [0] * len(gens)
        w = F(1)
        zsum = [F(0)] * s
        for ti in tup:
            combo, z = tiles[ti]
            for j in combo:
                mult[j] += 1
            w *= dets[combo]
            zsum = [a + b for a, b in zip(zsum, z)]
        shift = tuple(zsum[d] - order * center[d] for d in range(s))
        key = (tuple(mult), shift)
        acc[key] = acc.get(key, F(0)) + w
    boxes = {}
    terms = []
    for (mult, shift), w in sorted(acc.items()):
        bx = boxes.get(mult)
        if bx is None:
            used = [i for i, m in enumerate(mult) if m]
            bx = BoxSpline([gens[i] for i in used], [mult[i] for i in used])
            boxes[mult] = bx
        terms.append(BoxTerm(w, bx, shift))
    out = BoxSum(s, terms)
    # support of V_k: the zonotope of every generator taken k times, centred at 0
    out.hull = (tuple(gens), tuple([order] * len(gens)), tuple(-order * c for c in center))
    # sum over the lattice whose Voronoi cell is Z(gens): the translates of chi_V tile space,
    # so sum_n (chi_V * V_{k-1})(x - n) = integral of V_{k-1} = vol(V)^(k-1), exactly
    out.lattice_sum = zonotope_volume(gens) ** (order - 1)
    return out


H = F(1, 4)
# BCC Voronoi cell (truncated octahedron): edges (1/4)(1, +-1, 0) and permutations
BCC_VORONOI_GENS = [(H, H, 0), (H, -H, 0), (H, 0, H), (H, 0, -H), (0, H, H), (0, H, -H)]
# FCC Voronoi cell (rhombic dodecahedron): edges (1/4)(+-1, +-1, +-1)
FCC_VORONOI_GENS = [(H, H, H), (H, -H, -H), (-H, H, -H), (-H, -H, H)]


def zonotope_volume(gens):
    s = len(gens[0])
    tot = F(0)
    for combo in itertools.combinations(range(len(gens)), s):
        B = tuple(tuple(F(gens[j][a]) for j in combo) for a in range(s))
        tot += abs(exact.det(B))
    return tot
