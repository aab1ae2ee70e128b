"""CPU tests of the stabilizer-symmetry rewrite (kernel form "sym")."""

import pytest

from paper_2102_08518_b200 import list_fixtures, load_fixture, load_space
from paper_2102_08518_b200.symmetry import check, symmetrize
from tests.conftest import GOLDEN

NAMES = [p.stem for p in sorted((GOLDEN / "spaces").glob("*.json"))]


@pytest.mark.parametrize("name", NAMES)
def test_symmetrized_polynomials_are_identical(name):
    sp = load_space(GOLDEN / "spaces" / f"{name}.json")
    for i, rp in enumerate(sp.ref_polys):
        sub = next(s for s in sp.subregions if s.psi_index == i)
        f = symmetrize(rp.poly, sub.stencil)
        if f is None:
            continue
        assert f.terms_after <= f.terms_before
        assert check(f, rp.poly, sub.stencil, trials=3)


def test_expected_reductions():
    sp = load_fixture("tricubic")
    f = symmetrize(sp.ref_polys[0].poly, sp.subregions[0].stencil)
    assert f.axes == (0, 1, 2) and f.terms_after == 512
    sp = load_fixture("bcc_box5")
    f = symmetrize(sp.ref_polys[0].poly, sp.subregions[0].stencil)
    assert f.axes == (2,) and f.terms_after < sp.ref_polys[0].poly.terms.__len__()
