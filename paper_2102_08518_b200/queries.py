"""Synthetic query streams for the benchmark configurations.

Both generators are *index-addressable*: query i of the global stream is a pure
function of (seed, i), so a rank can generate exactly its shard [lo, hi) of the
same global set on its own device (multi-GPU runs see identical work).

* uniform:  x_i = E * hash(seed, i, axis) / 2^24, uniform in the periodic box.
* rays:     orthographic volume-rendering order: a W x H image of rays covering
            the projection of the box [0, E)^3, `steps` equispaced samples per ray
            over the box chord; query index ((tile * steps + step) * 32 + lane) with
            8 x 4-pixel warp tiles, so a warp samples 32 neighbouring rays at one
            depth and consecutive warps march along the rays.
"""

from __future__ import annotations


import numpy as np

_M1 = 0x9E3779B97F4A7C15
_M2 = 0xBF58476D1CE4E5B9
_M3 = 0x94D049BB133111EB


def _u64(v):
    """Wrap a Python int to a signed int64 constant (torch int64 arithmetic wraps)."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= 1 << 63 else v


def _mix(x):
    """splitmix64 finalizer on an int64 torch tensor (wrap-around arithmetic)."""
    import torch
    x = x ^ ((x >> 30) & ((1 << 34) - 1))
    x = x * _u64(_M2)
    x = x ^ ((x >> 27) & ((1 << 37) - 1))
    x = x * _u64(_M3)
    x = x ^ ((x >> 31) & ((1 << 33) - 1))
    return x


def uniform(lo: int, hi: int, extents, seed: int, device):
    """Queries [lo, hi) of the global uniform stream: (hi-lo, s) float32 on device."""
    import torch
    s = len(extents)
    idx = torch.arange(lo, hi, dtype=torch.int64, device=device)
    out = torch.empty((hi - lo, s), dtype=torch.float32, device=device)
    for d in range(s):
        key = idx * s + d + _u64(seed * _M1)
        r = _mix(key)
        u = ((r >> 40) & ((1 << 24) - 1)).to(torch.float32) * (1.0 / (1 << 24))
        out[:, d] = u * float(extents[d])
    return out


def camera(seed: int = 2):
    rng = np.random.default_rng(seed)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    up = rng.normal(size=3)
    up -= d * (up @ d)
    up /= np.linalg.norm(up)
    right = np.cross(d, up)
    return d, up, right


def rays(lo: int, hi: int, extents, width: int, height: int, steps: int, seed: int, device):
    """Queries [lo, hi) of the ray-ordered stream (width*height*steps queries in total)."""
    import torch
    E = np.array(extents, dtype=np.float64)
    d, up, right = camera(seed)
    center = E / 2
    corners = np.array([[x, y, z] for x in (0, E[0]) for y in (0, E[1]) for z in (0, E[2])])
    pr = (corners - center) @ right
    pu = (corners - center) @ up
    r0, r1 = pr.min(), pr.max()
    u0, u1 = pu.min(), pu.max()
    half = float(np.linalg.norm(E)) / 2
    idx = torch.arange(lo, hi, dtype=torch.int64, device=device)
    lane = idx % 32
    rest = idx // 32
    step = rest % steps
    tile = rest // steps
    tiles_x = width // 8
    tx = tile % tiles_x
    ty = tile // tiles_x
    px = tx * 8 + lane % 8
    py = ty * 4 + lane // 8
    f64 = torch.float64
    a = r0 + (px.to(f64) + 0.5) * ((r1 - r0) / width)
    b = u0 + (py.to(f64) + 0.5) * ((u1 - u0) / height)
    cen = torch.tensor(center, dtype=f64, device=device)
    dv = torch.tensor(d, dtype=f64, device=device)
    rv = torch.tensor(right, dtype=f64, device=device)
    uv = torch.tensor(up, dtype=f64, device=device)
    origin = cen[None, :] + a[:, None] * rv[None, :] + b[:, None] * uv[None, :]   # on the mid plane
    # box chord along d (slab test); rays that miss use the bounding-sphere chord
    inv = 1.0 / dv
    t1 = (0.0 - origin) * inv[None, :]
    t2 = (torch.tensor(E, dtype=f64, device=device)[None, :] - origin) * inv[None, :]
    tmin = torch.minimum(t1, t2).max(dim=1).values
    tmax = torch.maximum(t1, t2).min(dim=1).values
    miss = tmax <= tmin
    tmin = torch.where(miss, torch.full_like(tmin, -half), tmin)
    tmax = torch.where(miss, torch.full_like(tmax, half), tmax)
    t = tmin + (step.to(f64) + 0.5) * (tmax - tmin) / steps
    pts = origin + t[:, None] * dv[None, :]
    return pts.to(torch.float32)


def ray_table(extents, width: int, height: int, steps: int, seed: int = 2):
    """Per-pixel rays of the orthographic camera used by `rays`, for the fused renderer:
    (width*height, 8) float32 rows (origin xyz, direction xyz, t0, dt) in 8 x 4-pixel
    warp-tile order (row i is pixel pixel_of(i)); sample j of a ray is at
    o + (t0 + (j + 1/2) dt) d, evaluated in float32."""
    E = np.array(extents, dtype=np.float64)
    d, up, right = camera(seed)
    center = E / 2
    corners = np.array([[x, y, z] for x in (0, E[0]) for y in (0, E[1]) for z in (0, E[2])])
    pr = (corners - center) @ right
    pu = (corners - center) @ up
    r0, r1 = pr.min(), pr.max()
    u0, u1 = pu.min(), pu.max()
    half = float(np.linalg.norm(E)) / 2
    px, py = pixel_of(np.arange(width * height), width)
    a = r0 + (px + 0.5) * ((r1 - r0) / width)
    b = u0 + (py + 0.5) * ((u1 - u0) / height)
    origin = center[None, :] + a[:, None] * right[None, :] + b[:, None] * up[None, :]
    with np.errstate(divide="ignore"):
        inv = 1.0 / d
    t1 = (0.0 - origin) * inv[None, :]
    t2 = (E[None, :] - origin) * inv[None, :]
    tmin = np.minimum(t1, t2).max(axis=1)
    tmax = np.maximum(t1, t2).min(axis=1)
    miss = tmax <= tmin
    tmin = np.where(miss, -half, tmin)
    tmax = np.where(miss, half, tmax)
    out = np.empty((width * height, 8), dtype=np.float32)
    out[:, 0:3] = origin
    out[:, 3:6] = d[None, :]
    out[:, 6] = tmin
    out[:, 7] = (tmax - tmin) / steps
    return out


def pixel_of(i, width: int):
    """(px, py) of row i of a tile-ordered per-pixel table (8 x 4-pixel warp tiles)."""
    i = np.asarray(i)
    lane = i % 32
    tile = i // 32
    tiles_x = width // 8
    return (tile % tiles_x) * 8 + lane % 8, (tile // tiles_x) * 4 + lane // 8


def ray_count(width, height, steps):
    return width * height * steps


def make(kind: str, lo: int, hi: int, extents, device, seed: int = 1, **kw):
    if kind == "uniform":
        return uniform(lo, hi, extents, seed, device)
    if kind == "rays":
        return rays(lo, hi, extents, kw["width"], kw["height"], kw["steps"], kw.get("cam_seed", 2),
                    device)
    raise ValueError(kind)

