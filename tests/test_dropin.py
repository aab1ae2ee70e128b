"""The reference-facing Python surface behaves like `splinegen`'s:
extent-free `generate(space, GenConfig)`, the reference's f64 default, fixture names,
adoption of real reference `SplineSpace` objects, and the reference harness's
`prog = generate(...); runner = lambda pts: interpret_batch(prog, pts, data)` loop
(pkg/src/splinegen/bench.py:110-124) driven through the CUDA path."""

import os
import sys
from collections import Counter
from pathlib import Path

import numpy as np
import pytest

from tests.conftest import GOLDEN
from tests.gpu_util import ATOL_F32, ATOL_F64, RTOL_F32, RTOL_F64, close, load_golden

REF_SRC = Path("/root/reference/pkg/src")


def _with_reference():
    if not REF_SRC.exists():
        pytest.skip("reference sources are only present in the build container")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import splinegen
    return splinegen


def test_generate_without_extents_is_extent_free():
    from paper_2102_08518_b200 import GenConfig, Program, ScheduleParams, generate
    space, _, _, _ = load_golden("zp")
    prog = generate(space, GenConfig(ScheduleParams(1, space.stencil_size)))
    assert isinstance(prog, Program)
    a, b = prog.specialize((8, 8)), prog.specialize((13, 5))
    assert a.extents == ((8, 8),) and b.extents == ((13, 5),)
    assert prog.specialize((8, 8)) is a          # specializations are cached


def test_genconfig_defaults_follow_the_reference():
    from paper_2102_08518_b200 import GenConfig, ScheduleParams
    p = ScheduleParams(1, 4)
    assert GenConfig(p).float_width == "f64"              # codegen.py:38-46
    assert GenConfig(p, mode="sorted").float_width == "f32"   # f32-only execution modes
    assert GenConfig(p, mode="binned").float_width == "f32"
    assert GenConfig(p, float_width="f32").float_width == "f32"


def test_counter_is_rejected_and_max_steps_validated():
    from paper_2102_08518_b200 import DataVolume, InterpreterError, interpret_batch
    space, _, z, arrays = load_golden("zp")
    data = DataVolume(arrays)
    with pytest.raises(InterpreterError, match="counter"):
        interpret_batch(space, z["uniform_xs"][:4], data, counter=Counter())
    with pytest.raises(InterpreterError, match="max_steps"):
        interpret_batch(space, z["uniform_xs"][:4], data, max_steps=0)


def test_reference_fixture_names_resolve(monkeypatch):
    from paper_2102_08518_b200 import load_fixture
    from paper_2102_08518_b200.model import REFERENCE_FIXTURES, serialize_space
    monkeypatch.setenv("SPLINEGPU_FIXTURES", str(GOLDEN / "spaces"))
    for name in REFERENCE_FIXTURES:
        sp = load_fixture(name)
        assert sp.name == name
        want, _, _, _ = load_golden(name)
        assert serialize_space(sp) == serialize_space(want)


def test_unknown_fixture_names_the_remedy(monkeypatch):
    from paper_2102_08518_b200 import load_fixture
    monkeypatch.delenv("SPLINEGPU_FIXTURES", raising=False)
    with pytest.raises(FileNotFoundError, match="no fixture named 'nope'"):
        load_fixture("nope")


def test_reference_fixtures_load_from_an_installed_splinegen(monkeypatch):
    sg = _with_reference()
    from paper_2102_08518_b200 import load_fixture
    from paper_2102_08518_b200.model import REFERENCE_FIXTURES, serialize_space
    monkeypatch.delenv("SPLINEGPU_FIXTURES", raising=False)
    for name in REFERENCE_FIXTURES:
        assert serialize_space(load_fixture(name)) == sg.serialize_space(sg.load_fixture(name))


def test_adopt_a_real_reference_space():
    """SplineSpace.adopt (model.py) on objects built by the reference's own parser."""
    sg = _with_reference()
    from paper_2102_08518_b200 import SplineSpace, generate, GenConfig, ScheduleParams
    from paper_2102_08518_b200.model import serialize_space
    for name in ("zp", "trilinear_voronoi", "halfgrid1d"):
        ref = sg.load_fixture(name)
        ours = SplineSpace.adopt(ref)
        assert isinstance(ours, SplineSpace)
        assert serialize_space(ours) == sg.serialize_space(ref)
        # and generate accepts the reference object directly
        prog = generate(ref, GenConfig(ScheduleParams(1, ours.stencil_size)), (6,) * ours.dim)
        assert prog.space.nsubregions == ours.nsubregions


def test_extension_spaces_validate_only_outside_strict_mode():
    from paper_2102_08518_b200.model import load_fixture, validate_space
    sp = load_fixture("fcc_voronoi3")        # per-polynomial stencil sizes 6..8
    assert not sp.uniform_stencils
    assert not [d for d in validate_space(sp) if d.severity == "error"]
    strict = [d for d in validate_space(sp, strict=True) if d.severity == "error"]
    assert [d.path for d in strict] == ["subregions"]


# -- GPU: the reference harness's loop shape through the CUDA path --------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["zp_k2", "trilinear_voronoi", "bcc_box_linear"])
@pytest.mark.parametrize("float_width", ["f64", "f32"])
def test_run_sweep_loop_shape(name, float_width):
    """bench.py:110-136 of the reference: one program per (m, d, mode) cell from the
    extent-free generate, a runner with the `runner(pts) -> (N,)` contract, the oracle
    spot-check at 1e-9 (f64) / 1e-3 (f32) -- here at the north star's 1e-12 / 1e-5."""
    from oracle import refeval
    from paper_2102_08518_b200 import DataVolume, GenConfig, ScheduleParams, generate, interpret_batch
    space, ospace, z, arrays = load_golden(name)
    dt = np.float64 if float_width == "f64" else np.float32
    data = DataVolume([a.astype(dt) for a in arrays])
    pts = z["uniform_xs"][:256].astype(np.float64)
    want = refeval.reference_eval_batch(ospace, pts.astype(dt).astype(np.float64),
                                        [a.astype(np.float64) for a in data.arrays])
    n = space.stencil_size
    rtol, atol = (RTOL_F64, ATOL_F64) if float_width == "f64" else (RTOL_F32, ATOL_F32)
    for m, d in [(1, n), (2, max(2, n // 2)), (n, n)]:
        for mode in ("predicated", "branchy"):
            prog = generate(space, GenConfig(ScheduleParams(m, d, mode), float_width=float_width))

            def runner(p, prog=prog):
                return interpret_batch(prog, p, data)
            got = runner(pts)
            assert got.dtype == dt and got.shape == (len(pts),)
            assert np.all(close(got, want, rtol, atol)), \
                (m, d, mode, float(np.abs(got.astype(np.float64) - want).max()))


@pytest.mark.gpu
def test_one_program_many_volumes_and_in_place_edits():
    from oracle import refeval
    from paper_2102_08518_b200 import DataVolume, GenConfig, ScheduleParams, generate, interpret_batch
    space, ospace, z, _ = load_golden("zp")
    prog = generate(space, GenConfig(ScheduleParams(1, space.stencil_size)))
    rng = np.random.default_rng(3)
    for ext in [(8, 8), (11, 7), (16, 16)]:
        data = DataVolume([rng.random(ext)])
        pts = rng.random((300, 2)) * np.array(ext)
        got = interpret_batch(prog, pts, data)
        want = refeval.reference_eval_batch(ospace, pts, list(data.arrays))
        assert np.abs(got - want).max() <= 1e-12
        data.arrays[0][...] = 1.0                 # edited in place: the next call must see it
        assert np.abs(interpret_batch(prog, pts, data) - 1.0).max() <= 1e-12


@pytest.mark.gpu
def test_evaluator_rejects_host_tensors():
    import torch
    from paper_2102_08518_b200 import Evaluator, GenConfig, InterpreterError, ScheduleParams
    space, _, z, arrays = load_golden("zp")
    ev = Evaluator(space, arrays, GenConfig(ScheduleParams(1, space.stencil_size), float_width="f32"))
    with pytest.raises(InterpreterError, match="CUDA tensor"):
        ev(torch.from_numpy(z["uniform_xs"][:8].copy()))
    xs = torch.from_numpy(z["uniform_xs"][:8].copy()).cuda()
    with pytest.raises(InterpreterError, match="CUDA tensor"):
        ev(xs, out=torch.empty(8))
