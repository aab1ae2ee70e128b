"""Pin the CPU oracle (oracle/refeval.py) to the reference's own outputs.

The vectors under tests/golden/ were produced by running the unmodified
reference package (tests/golden/make_golden.py).  The oracle must reproduce
them bit-for-bit: values (float64), lattice shifts k and sub-region indices.
"""

import json

import numpy as np
import pytest

from oracle import refeval
from tests.conftest import GOLDEN

NAMES = sorted(p.stem for p in (GOLDEN / "spaces").glob("*.json"))
SETS = ("uniform", "grid", "adversarial")


def _load(name):
    space = refeval.load_space_file(GOLDEN / "spaces" / f"{name}.json")
    z = np.load(GOLDEN / f"{name}.npz")
    arrays = [z[f"vol_{i}"].astype(np.float64) for i in range(space.ncosets)]
    return space, z, arrays


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("which", SETS)
def test_oracle_values_bit_exact(name, which):
    space, z, arrays = _load(name)
    xs = z[f"{which}_xs"].astype(np.float64)
    got = refeval.reference_eval_batch(space, xs, arrays)
    want = z[f"{which}_value"]
    assert np.array_equal(got, want), float(np.abs(got - want).max())


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("which", SETS)
def test_oracle_selection_bit_exact(name, which):
    space, z, _ = _load(name)
    xs = z[f"{which}_xs"].astype(np.float64)
    sel = refeval.selection(space, xs)
    for ci, (k, sub) in enumerate(sel):
        assert np.array_equal(k, z[f"{which}_k"][ci])
        assert np.array_equal(sub, z[f"{which}_sub"][ci])


@pytest.mark.parametrize("name", NAMES)
def test_reference_generated_code_agrees(name):
    """The reference's own f64 generated program agrees with its oracle (1e-9)."""
    space, z, arrays = _load(name)
    if "uniform_interp_f64" not in z:
        pytest.skip("extension space: the reference generator refuses it (make_golden.py)")
    want = z["uniform_value"]
    got = z["uniform_interp_f64"]
    assert np.all(np.abs(got - want) <= 1e-12 + 1e-9 * np.maximum(abs(got), abs(want)))


def test_falg_recorded_for_every_space():
    falg = json.loads((GOLDEN / "falg.json").read_text())
    for name in NAMES:
        assert falg[name] > 0


def test_partition_of_unity_zp():
    space = refeval.load_space_file(GOLDEN / "spaces" / "zp.json")
    rng = np.random.default_rng(0)
    pts = rng.random((1000, 2)) * 8
    got = refeval.reference_eval_batch(space, pts, [np.ones((8, 8))])
    assert np.abs(got - 1.0).max() <= 1e-12


def test_convolution_matches_reference_eval():
    space = refeval.load_space_file(GOLDEN / "spaces" / "zp.json")
    rng = np.random.default_rng(7)
    vol = [rng.random((8, 8))]
    pts = rng.random((300, 2)) * 8
    a = refeval.reference_eval_batch(space, pts, vol)
    b = refeval.convolution_eval_batch(space, pts, vol)
    assert np.all(np.abs(a - b) <= 1e-12 + 1e-9 * np.maximum(abs(a), abs(b)))


def test_gradient_matches_central_difference():
    space = refeval.load_space_file(GOLDEN / "spaces" / "zp.json")
    rng = np.random.default_rng(9)
    vol = [rng.random((8, 8))]
    pts = rng.random((200, 2)) * 8
    _, g = refeval.reference_eval_batch(space, pts, vol, grad=True)
    h = 1e-6
    for d in range(2):
        e = np.zeros(2)
        e[d] = h
        fd = (refeval.reference_eval_batch(space, pts + e, vol)
              - refeval.reference_eval_batch(space, pts - e, vol)) / (2 * h)
        assert np.abs(fd - g[:, d]).max() <= 1e-5


def test_unreachable_sigma_raises():
    import dataclasses
    space = refeval.load_space_file(GOLDEN / "spaces" / "zp.json")
    bad = dataclasses.replace(space, sigma=(-1,) + space.sigma[1:])
    q0 = np.array([[0.1, 0.3]])  # x0 - x1 < 0, x0 + x1 >= 0 -> q = 2
    with pytest.raises(refeval.UnreachableRegionError):
        # find a point landing in q == 0: x0 < x1 and x0 < -x1
        refeval.reference_eval_batch(bad, np.array([[-0.3, 0.1]]), [np.ones((8, 8))])
    refeval.reference_eval_batch(bad, q0, [np.ones((8, 8))])
