"""Fused renderer: ray tables and the compositing oracle on CPU; the
sg_render kernel against the oracle on the GPU (bit-identical sample positions, values
from the restated reference evaluator, fp64 compositing)."""

import numpy as np
import pytest

from oracle import refeval
from oracle import render as orender
from paper_2102_08518_b200.queries import pixel_of, ray_table
from tests.gpu_util import load_golden


def test_ray_table_covers_the_box():
    E = (20, 20, 20)
    rays = ray_table(E, 16, 8, 32)
    assert rays.shape == (128, 8) and rays.dtype == np.float32
    pos = orender.sample_positions(rays, 32)
    inside = ((pos >= -1e-3) & (pos <= 20 + 1e-3)).all(axis=2)
    half = float(np.linalg.norm(E)) / 2
    hit = np.abs(rays[:, 6] + half) > 1e-3        # rays that miss march the sphere chord
    assert hit.mean() > 0.8 and inside[hit].all()
    px, py = pixel_of(np.arange(128), 16)
    assert sorted(zip(px.tolist(), py.tolist())) == [(x, y) for x in range(16) for y in range(8)]


def test_oracle_composite_limits():
    space, ospace, z, arrays = load_golden("trilinear")
    E = arrays[0].shape
    rays = ray_table(E, 8, 4, 8)
    clear = np.array([10.0, 1.0, 1.0, 1, 1, 1, 1, 1, 1, 1, 0, 0], dtype=np.float32)  # f_lo above data
    img = orender.render(ospace, arrays, rays, 8, clear)
    assert np.abs(img).max() == 0.0
    opaque = np.array([-10.0, 0.05, 1e9, 1, 0, 0, 1, 0, 0, 1, 0, 0], dtype=np.float32)
    img = orender.render(ospace, arrays, rays, 8, opaque)
    assert np.allclose(img[:, 3], 1.0) and np.allclose(img[:, 0], 1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["bcc_voronoi2", "bcc_box5", "fcc_box6", "tricubic", "fcc_voronoi2"])
@pytest.mark.parametrize("shade", [False, True])
@pytest.mark.parametrize("variant", ["march", "sorted"])
def test_render_matches_oracle(name, shade, variant):
    import torch
    from paper_2102_08518_b200.render import Renderer
    space, ospace, z, arrays = load_golden(name)
    kw = dict(block=128, tile=512) if variant == "sorted" else dict(block=128, tile=0)
    # 16 x 8 pixels = one 128-ray block; 24 steps = 6 chunks of 4 steps in the sorted kernel
    r = Renderer(space, arrays, 16, 8, 24, shade=shade, **kw)
    img = r().cpu().numpy().reshape(-1, 4)
    want = orender.render(ospace, arrays, r.rays_np, 24, r.tf_np, shade=shade)
    px, py = pixel_of(np.arange(16 * 8), 16)
    want_img = np.zeros((8, 16, 4))
    want_img[py, px] = want
    err = np.abs(img - want_img.reshape(-1, 4)).max()
    assert err <= 2e-5, err
    assert want_img[..., 3].max() > 0.05      # the test image is not empty


@pytest.mark.gpu
def test_render_rejects_eval_and_vice_versa():
    import torch
    from paper_2102_08518_b200 import runtime
    from paper_2102_08518_b200.render import Renderer
    space, ospace, z, arrays = load_golden("zp_k2") if False else load_golden("trilinear")
    r = Renderer(space, arrays, 8, 4, 4)
    xs = torch.zeros((4, 3), dtype=torch.float32, device="cuda")
    out = torch.empty(4, device="cuda")
    with pytest.raises(runtime.SplineGpuError):
        runtime.eval_device(r.ev.module, r.ev.volume, xs, out)


@pytest.mark.gpu
def test_render_full_size_constant_volume_closed_form():
    """Bench-size render (512 x 512 x 256, the sorted tiles) of an all-ones volume: f = 1 at
    every sample (partition of unity), so each ray composites a constant opacity
    a = min(opacity * dt, 1): A = 1 - (1 - a)^steps, rgb = rgb_hi * A."""
    from paper_2102_08518_b200 import load_fixture
    from paper_2102_08518_b200.render import DEFAULT_TF, Renderer
    space = load_fixture("bcc_voronoi2")
    E = (203, 203, 203)
    ones = [np.ones(E, dtype=np.float32) for _ in range(space.ncosets)]
    r = Renderer(space, ones, 512, 512, 256)
    img = r().cpu().numpy().reshape(-1, 4)
    px, py = pixel_of(np.arange(512 * 512), 512)
    dt = np.zeros((512, 512))
    dt[py, px] = r.rays_np[:, 7]
    a = np.minimum(DEFAULT_TF["opacity"] * dt.astype(np.float64), 1.0).reshape(-1)
    A = 1.0 - (1.0 - a) ** 256
    assert np.abs(img[:, 3] - A).max() <= 2e-4
    for ch in range(3):
        assert np.abs(img[:, ch] - DEFAULT_TF["rgb_hi"][ch] * A).max() <= 2e-4
