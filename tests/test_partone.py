"""The Part-I producer (partone/) reproduces the reference's shipped spaces and
builds valid spaces for the benchmark splines (CPU only)."""

from fractions import Fraction as F

import numpy as np
import pytest

from oracle import refeval
from paper_2102_08518_b200 import list_fixtures, load_fixture, serialize_space, validate_space
from paper_2102_08518_b200.partone.boxspline import BoxSpline, centered_box
from paper_2102_08518_b200.partone.producer import Producer
from paper_2102_08518_b200.partone.tensor import bspline_pieces
from tests.conftest import GOLDEN

I1, I2, I3 = [[1]], [[1, 0], [0, 1]], [[1, 0, 0], [0, 1, 0], [0, 0, 1]]
SHIPPED = {
    "linear1d": (centered_box([(1,)], [2]), [(0,)], I1, "floor", (16,)),
    "halfgrid1d": (centered_box([(F(1, 2),)], [2]), [(0,), (F(1, 2),)], [[F(1, 2)]], "floor", (16,)),
    "zp": (centered_box([(1, 0), (0, 1), (1, 1), (1, -1)]), [(0, 0)], I2, "round_nearest", (8, 8)),
    "trilinear": (centered_box([(1, 0, 0), (0, 1, 0), (0, 0, 1)], [2, 2, 2]), [(0, 0, 0)], I3,
                  "floor", (6, 6, 6)),
    "trilinear_voronoi": (centered_box([(1, 0, 0), (0, 1, 0), (0, 0, 1)], [2, 2, 2]), [(0, 0, 0)],
                          I3, "round_nearest", (6, 6, 6)),
}


def test_box_spline_recurrence_matches_cardinal_bspline():
    b = BoxSpline([(1,)], [4])
    pieces = bspline_pieces(3)
    for x in (F(1, 3), F(13, 7), F(5, 2), F(37, 10)):
        j = int(x)
        u = x - j
        assert b((x,)) == sum(c * u ** e for e, c in enumerate(pieces[j]))


def test_zp_box_spline_matches_reference_basis():
    ospace = refeval.load_space_file(GOLDEN / "spaces" / "zp.json")
    phi = centered_box([(1, 0), (0, 1), (1, 1), (1, -1)])
    rng = np.random.default_rng(1)
    ys = [(F(int(a), 97), F(int(b), 89)) for a, b in rng.integers(-190, 190, size=(40, 2))]
    want = refeval.basis_from_delta_batch(ospace, np.array([[float(a), float(b)] for a, b in ys]))
    got = np.array([float(phi(y)) for y in ys])
    assert np.abs(got - want).max() <= 1e-15


@pytest.mark.parametrize("name", sorted(SHIPPED))
def test_producer_reproduces_shipped_fixture(name):
    phi, cos, gen, rnd, ext = SHIPPED[name]
    sp = Producer(phi, cos, gen, name, rnd).run()
    assert not [d for d in validate_space(sp) if d.severity == "error"]
    mine = refeval.load_space(serialize_space(sp))
    ref = refeval.load_space_file(GOLDEN / "spaces" / f"{name}.json")
    rng = np.random.default_rng(3)
    arr = [rng.random(ext) for _ in cos]
    xs = rng.random((2000, len(ext))) * np.array(ext)
    a = refeval.reference_eval_batch(mine, xs, arr)
    b = refeval.reference_eval_batch(ref, xs, arr)
    assert np.abs(a - b).max() <= 1e-13


@pytest.mark.parametrize("name", ["tricubic", "bcc_box5", "bcc_box_linear", "fcc_box6"])
def test_shipped_space_partition_of_unity_and_linear_reproduction(name):
    sp = load_fixture(name)
    osp = refeval.load_space_file(GOLDEN / "spaces" / f"{name}.json")
    ext = (8, 8, 8)
    rng = np.random.default_rng(5)
    xs = rng.random((500, 3)) * 8
    ones = [np.ones(ext) for _ in range(sp.ncosets)]
    assert np.abs(refeval.reference_eval_batch(osp, xs, ones) - 1).max() <= 1e-12
    # linear precision: data = x0 coordinate of each lattice site (away from the wrap)
    arrs = []
    for c in sp.lattice.cosets:
        g = np.indices(ext).astype(np.float64)
        arrs.append(g[0] + float(c[0]))
    inner = 3 + rng.random((300, 3)) * 2
    got = refeval.reference_eval_batch(osp, inner, arrs)
    assert np.abs(got - inner[:, 0]).max() <= 1e-11


def test_bcc_box5_structure():
    sp = load_fixture("bcc_box5")
    assert sp.ncosets == 2 and sp.nref == 1 and sp.nsubregions == 24 and sp.stencil_size == 16
    assert len(sp.planes) == 6


@pytest.mark.parametrize("name", ["bcc_box5", "fcc_box6"])
def test_shipped_space_symmetry(name):
    """phi(g y) == phi(y) for a signed permutation g, through the tables (oracle)."""
    osp = refeval.load_space_file(GOLDEN / "spaces" / f"{name}.json")
    rng = np.random.default_rng(8)
    ys = rng.uniform(-1.5, 1.5, size=(200, 3))
    a = refeval.basis_from_delta_batch(osp, ys)
    b = refeval.basis_from_delta_batch(osp, ys[:, [2, 0, 1]] * np.array([-1, 1, -1]))
    assert np.abs(a - b).max() <= 1e-12


def test_fixture_listing():
    names = list_fixtures()
    for n in ("tricubic", "bcc_box5"):
        assert n in names
