"""Fused volume renderer: the consumer of the evaluation path.

The paper's application is volume rendering: rays are marched through
the coefficient lattice and the spline is reconstructed at every sample.  Here ray
setup, reconstruction (+ gradient for shading) and front-to-back compositing run in
ONE generated sm_100a kernel (GenConfig.mode = "render", C ABI `sg_render`), so the
2^26 sample positions and values of a 512 x 512 x 256 march never round-trip through
HBM as they do in the unfused query/result path (bench config c3).

Transfer function (12 floats, `tf`): density d = clamp((f - f_lo) / (f_hi - f_lo), 0, 1);
opacity per sample a = min(d * opacity * dt, 1); colour = lerp(rgb_lo, rgb_hi, d),
times a Lambert factor 0.3 + 0.7 |g . L| / |g| when shading (g = grad f);
C += (1 - A) a colour, A += (1 - A) a.
"""

from __future__ import annotations

import numpy as np

from . import runtime
from .api import Evaluator
from .cudagen import GenConfig, generate
from .model import SplineSpace
from .queries import pixel_of, ray_table
from .schedule import ScheduleParams

DEFAULT_TF = dict(f_lo=0.3, f_hi=0.7, opacity=0.02, rgb_lo=(0.1, 0.2, 0.9), rgb_hi=(1.0, 0.4, 0.1),
                  light=(1.0, 1.0, 1.0))


def tf_vector(f_lo, f_hi, opacity, rgb_lo, rgb_hi, light):
    L = np.asarray(light, dtype=np.float64)
    L = L / np.linalg.norm(L)
    return np.array([f_lo, 1.0 / (f_hi - f_lo), opacity, *rgb_lo, *rgb_hi, *L], dtype=np.float32)


def render_config(space: SplineSpace, shade: bool = False, **variant) -> GenConfig:
    """The renderer's kernel variant.  One ray per thread (predicated dispatch, immediates,
    128-thread CTAs) for single-polynomial spaces; for K > 1 reference polynomials the
    samples of 128 rays x (tile / 128) steps are sorted by psi in shared memory first
    (measured on B200: BCC Voronoi 2.75 -> 2.18 ms per 512 x 512 x 256 image)."""
    kw = dict(params=ScheduleParams(1, space.stencil_size, "predicated"), mode="render",
              grad=shade, block=128)
    if len(space.ref_polys) > 1:
        big = sum(len(rp.poly.terms) for rp in space.ref_polys) > 4000
        if big and shade:
            # value + gradient of large polynomials: coefficient tables in shared memory and
            # one site loop for all of them (the gradient comes from the same monomial sums);
            # per-polynomial immediate code (x4 with the derivatives) overflows the I-cache
            kw.update(block=384, tile=768, coeffs="table", tloop=1)
        elif big:
            # immediates, warp chunks handed out in polynomial order (cmajor=3): measured on
            # B200 for the order-3 BCC Voronoi spline, 45.0 -> 10.5 ms per 512 x 512 x 256
            kw.update(block=512, tile=3072, cmajor=3, min_blocks=1)
        else:
            kw.update(block=256, tile=1024) if shade else kw.update(block=512, tile=1536)
        kw.update(radix=1)   # sub-region from the plane-family counts when they cover every plane
    kw.update(variant)
    return GenConfig(**kw)


class Renderer:
    """Render `width x height` images of a coefficient volume with `steps` samples per ray."""

    def __init__(self, space: SplineSpace, arrays, width: int, height: int, steps: int,
                 cam_seed: int = 2, shade: bool = False, tf: dict | None = None, device: int = 0,
                 **variant):
        import torch
        if width % 8 or height % 4:
            raise ValueError("width must be a multiple of 8 and height of 4 (warp tiles)")
        arrays = arrays.arrays if hasattr(arrays, "arrays") else list(arrays)
        extents = tuple(int(e) for e in arrays[0].shape)
        self.prog = generate(space, render_config(space, shade, **variant), tuple(extents))
        self.ev = Evaluator(space, arrays, prog=self.prog, device=device)
        self.width, self.height, self.steps = width, height, steps
        self.dev = torch.device("cuda", device)
        self.rays_np = ray_table(tuple(extents), width, height, steps, cam_seed)
        self.rays = torch.from_numpy(self.rays_np).to(self.dev)
        self.tf_np = tf_vector(**(tf or DEFAULT_TF))
        self.tf = torch.from_numpy(self.tf_np).to(self.dev)
        self.rgba = torch.empty((width * height, 4), dtype=torch.float32, device=self.dev)
        px, py = pixel_of(np.arange(width * height), width)
        self._order = torch.from_numpy(py * width + px).to(self.dev)

    @property
    def samples(self) -> int:
        return self.width * self.height * self.steps

    def launch(self, stream=None):
        """Render into self.rgba (tile order), asynchronously on `stream`."""
        runtime.render_device(self.ev.module, self.ev.volume, self.rays, self.steps, self.tf,
                              self.rgba, stream)
        return self.rgba

    def __call__(self, stream=None):
        """(height, width, 4) image on the device."""
        import torch
        rgba = self.launch(stream)
        img = torch.empty_like(rgba)
        img[self._order] = rgba
        self.ev.module.status()
        return img.view(self.height, self.width, 4)
