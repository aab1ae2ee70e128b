"""Adversarial query sets for bit-exact selection tests (not collected: no test_ prefix).

`adversarial_points` is the generator tests/golden/make_golden.py used for the golden
vectors (moved here so the GPU tests can scale it to the benchmark extents without
importing the reference): k + 1/2 +- 1 ulp(f32), |x| < 1e-9 next to coset offsets,
points exactly on BSP planes (where `>=` decides), and points outside [0, E).
`border_points` adds the binned kernels' own hazards: queries within an ulp of bin
edges (the f32 binning may put them one bin off), at 0 and E - ulp (periodic wrap).
"""

from __future__ import annotations

import numpy as np


def _f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def adversarial_points(space, extents, rng, count):
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
            ax = int(np.argmax(np.abs(nrm)))
            rest = loc @ nrm - nrm[ax] * loc[:, ax]
            loc[:, ax] = (float(plane.offset) - rest) / nrm[ax]
            cand = site + loc
            ok = np.all(np.abs(cand - np.round(cand * 64) / 64) == 0, axis=1)
            pts.append(cand[ok])
    # 4) out-of-range (negative and beyond the extent)
    pts.append(_f32((rng.random((per, s)) - 0.5) * 4 * e))
    return _f32(np.concatenate(pts, axis=0))


def border_points(extents, bin_, rng, count):
    """Queries within one f32 ulp of bin edges (multiples of `bin_` cells, 0 = none), of
    0 and of E on random axes; the other coordinates uniform."""
    e = np.array(extents, dtype=np.float64)
    s = len(extents)
    pts = rng.random((count, s)) * e
    edges = [np.array([0.0, e[d]]) for d in range(s)]
    if bin_:
        edges = [np.concatenate([np.arange(0, e[d], bin_), [e[d]]]) for d in range(s)]
    for i in range(count):
        for d in rng.choice(s, size=rng.integers(1, s + 1), replace=False):
            v = np.float32(rng.choice(edges[d]))
            step = rng.integers(-2, 3)
            for _ in range(abs(step)):
                v = np.nextafter(v, np.float32(np.inf if step > 0 else -np.inf))
            pts[i, d] = float(v)
    return _f32(pts)
