"""Tensor-product B-spline spaces on Z^s (config C1: tricubic on Z^3).

Floor region of evaluation (x_loc in [0,1)^s), one sub-region, identity
transform; the stencil is {-(p-1)//2 .. } ^ s in C order (last axis fastest)
so consecutive data symbols are contiguous in memory.  Same construction
pattern as the reference's `_tensor_linear` fixture builder
(pkg/scripts/make_fixtures.py:183-193), generalised to degree p.
"""

from __future__ import annotations

import itertools
from fractions import Fraction

from .. import exact
from ..model import (BspPlane, LatticeSpec, RefPoly, RegionMap, SplineSpace, SubRegion,
                     SubRegionIndexer)
from ..poly import Poly


def bspline_pieces(p: int):
    """Uniform B-spline of degree p on knots 0..p+1, built exactly by repeated
    convolution with the unit box: pieces[j] is B_p on [j, j+1) as coefficients
    of u = t - j (lowest degree first)."""
    pieces = [[Fraction(1)]]
    for deg in range(1, p + 1):
        new = []
        for j in range(deg + 1):
            # B_deg(j + u) = int_u^1 B_{deg-1}|_{j-1}(v) dv + int_0^u B_{deg-1}|_j(v) dv
            poly = [Fraction(0)] * (deg + 1)
            if j >= 1:
                for e, a in enumerate(pieces[j - 1]):
                    poly[0] += a / (e + 1)
                    poly[e + 1] -= a / (e + 1)
            if j < len(pieces):
                for e, a in enumerate(pieces[j]):
                    poly[e + 1] += a / (e + 1)
            new.append(poly)
        pieces = new
    return pieces


def weights_1d(p: int):
    """[(site offset o, weight polynomial in u)] for x = k + u, u in [0,1).

    The centered B-spline of odd degree p is supported on [-(p+1)/2, (p+1)/2];
    site k + o contributes B_p(u - o + (p+1)/2), i.e. piece (p+1)/2 - o."""
    if p % 2 == 0:
        raise ValueError("floor-ROE tensor spaces are built for odd degrees")
    pieces = bspline_pieces(p)
    half = (p + 1) // 2
    return [(o, pieces[half - o]) for o in range(-(half - 1), half + 1)]


def tensor_bspline(dim: int, p: int, name: str | None = None) -> SplineSpace:
    w = weights_1d(p)
    sites = list(itertools.product(range(len(w)), repeat=dim))
    terms = {}
    for j, idx in enumerate(sites):
        # product of 1-D polynomials, expanded
        polys = [w[i][1] for i in idx]
        for exps in itertools.product(*[range(len(pp)) for pp in polys]):
            coeff = Fraction(1)
            for pp, e in zip(polys, exps):
                coeff *= pp[e]
            if coeff:
                key = (tuple(exps), j)
                terms[key] = terms.get(key, Fraction(0)) + coeff
    poly = Poly(dim, terms)
    stencil = tuple(tuple(w[i][0] for i in idx) for idx in sites)
    I = exact.eye(dim)
    zero = tuple(Fraction(0) for _ in range(dim))
    return SplineSpace(
        name=name or f"tensor_deg{p}_{dim}d",
        dim=dim,
        lattice=LatticeSpec(generator=I, cosets=(zero,)),
        region_map=RegionMap(shape="parallelepiped", rounding="floor", basis=I),
        planes=(),
        indexer=SubRegionIndexer(modulus=1, sigma=(0,)),
        subregions=(SubRegion(transform=I, shift=zero, stencil=stencil, psi_index=0),),
        ref_polys=(RefPoly(poly),),
    )


def tricubic() -> SplineSpace:
    return tensor_bspline(3, 3, "tricubic")
