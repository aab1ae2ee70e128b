"""CPU tests: index-addressable query streams and symbolic box-spline pieces."""

from fractions import Fraction as F

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2102_08518_b200 import queries  # noqa: E402
from paper_2102_08518_b200.partone.boxspline import centered_box  # noqa: E402
from paper_2102_08518_b200.partone.pieces import PieceEvaluator, peval, phi_piece  # noqa: E402
from paper_2102_08518_b200.partone.voronoi import (BCC_VORONOI_GENS, FCC_VORONOI_GENS,  # noqa: E402
                                                   voronoi_spline, zonotope_tiles,
                                                   zonotope_volume)


def test_uniform_stream_is_index_addressable():
    full = queries.uniform(0, 4096, (101, 101, 101), 1, "cpu")
    part = queries.uniform(1000, 3000, (101, 101, 101), 1, "cpu")
    assert torch.equal(full[1000:3000], part)
    assert float(full.min()) >= 0 and float(full.max()) < 101
    assert abs(float(full.mean()) - 50.5) < 2.0


def test_ray_stream_is_index_addressable_and_coherent():
    full = queries.rays(0, 32 * 64 * 8, (203, 203, 203), 64, 64, 8, 2, "cpu")
    part = queries.rays(96, 160, (203, 203, 203), 64, 64, 8, 2, "cpu")
    assert torch.equal(full[96:160], part)
    warp = full[:32]
    assert float((warp.max(0).values - warp.min(0).values).max()) < 30.0


def test_symbolic_pieces_equal_point_values():
    h = F(1, 2)
    phi = centered_box([(h, h, h), (h, -h, -h), (-h, h, -h), (-h, -h, h)], [2, 2, 2, 2])
    ev = PieceEvaluator(3)
    p = (F(1, 7), F(2, 19), F(-3, 37))
    for site in [(0, 0, 0), (1, 0, 0), (0, 1, -1)]:
        P = phi_piece(phi, ev, p, site)
        for x in [p, (F(1, 7) + F(1, 1000), F(2, 19), F(-3, 37) - F(1, 2000))]:
            assert peval(P, x) == phi(tuple(a - b for a, b in zip(x, site)))


@pytest.mark.parametrize("gens,vol", [(BCC_VORONOI_GENS, F(1, 2)), (FCC_VORONOI_GENS, F(1, 4))])
def test_voronoi_cell_tiling(gens, vol):
    assert zonotope_volume(gens) == vol            # 1 / lattice density
    phi1 = voronoi_spline(gens, 1)                  # the cell's indicator
    rng = np.random.default_rng(0)
    for _ in range(60):
        x = tuple(F(int(v), 1000) for v in rng.integers(-520, 520, size=3))
        assert phi1(x) in (0, 1)
    tiles = zonotope_tiles(gens)
    assert len(tiles) == (16 if len(gens) == 6 else 4)
