"""CPU oracle for the fused renderer -- TEST INFRASTRUCTURE ONLY.

Restates, in numpy float64, what `sg_render` computes: sample positions formed in
float32 exactly as the kernel forms them (t = t0 + (j + 1/2) dt, p = o + t d, each
operation rounded to float32, no fused multiply-add), the spline value (and gradient)
at every sample from `refeval.reference_eval_batch` (the restatement of the reference
evaluator, pkg/src/splinegen/oracle.py:77-104), and front-to-back compositing with the
transfer function documented in paper_2102_08518_b200/render.py.  Only tests/ may use it.
"""

from __future__ import annotations

import numpy as np

from . import refeval


def sample_positions(rays: np.ndarray, steps: int) -> np.ndarray:
    """(npix, steps, 3) float32 sample positions, bit-identical to the kernel's."""
    rays = np.asarray(rays, dtype=np.float32)
    o, d = rays[:, None, 0:3], rays[:, None, 3:6]
    t0, dt = rays[:, None, 6:7], rays[:, None, 7:8]
    j = np.arange(steps, dtype=np.float32)[None, :, None]
    t = (t0 + (j + np.float32(0.5)) * dt).astype(np.float32)
    return (o + t * d).astype(np.float32)


def render(space: refeval.OSpace, arrays, rays: np.ndarray, steps: int, tf: np.ndarray,
           shade: bool = False) -> np.ndarray:
    """(npix, 4) float64 premultiplied rgba in the rays' (tile) order."""
    tf = np.asarray(tf, dtype=np.float64)
    f_lo, inv, op = tf[0], tf[1], tf[2]
    c_lo, c_hi, L = tf[3:6], tf[6:9], tf[9:12]
    pos = sample_positions(rays, steps)
    npix = pos.shape[0]
    flat = pos.reshape(-1, 3).astype(np.float64)
    arrays = [np.asarray(a, dtype=np.float64) for a in arrays]
    if shade:
        f, g = refeval.reference_eval_batch(space, flat, arrays, grad=True)
        g = g.reshape(npix, steps, 3)
    else:
        f = refeval.reference_eval_batch(space, flat, arrays)
    f = f.reshape(npix, steps)
    dt = np.asarray(rays, dtype=np.float64)[:, 7]
    C = np.zeros((npix, 3))
    A = np.zeros(npix)
    for j in range(steps):
        dn = np.clip((f[:, j] - f_lo) * inv, 0.0, 1.0)
        al = np.minimum(dn * op * dt, 1.0)
        if shade:
            gj = g[:, j]
            gl = np.sqrt((gj * gj).sum(axis=1))
            sh = np.where(gl > 0, 0.3 + 0.7 * np.abs(gj @ L) / np.where(gl > 0, gl, 1.0), 1.0)
        else:
            sh = 1.0
        w = (1.0 - A) * al * sh
        C += w[:, None] * (c_lo[None, :] + dn[:, None] * (c_hi - c_lo)[None, :])
        A += (1.0 - A) * al
    return np.concatenate([C, A[:, None]], axis=1)
