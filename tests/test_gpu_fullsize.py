"""Parity at the benchmark configurations' full sizes (needs a B200).

Size-independent properties on the full volumes and query streams of bench.py's
configs (partition of unity, linearity in the data, periodic shift invariance),
plus an oracle spot check on a subsample of the same workload.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import bench  # noqa: E402
from oracle import refeval  # noqa: E402
from paper_2102_08518_b200 import Evaluator  # noqa: E402
from paper_2102_08518_b200.model import SPACES_DIR  # noqa: E402

pytestmark = pytest.mark.gpu

CFGS = ["c1", "c2", "c3", "c4", "c4v", "c4v4", "c5", "c5u"]
NQ = 1 << 20


def _setup(cfg, ones=False):
    dev = torch.device("cuda", 0)
    space, arrays, _ = bench.make_inputs(cfg, 0, dev)
    xs = bench.make_queries(cfg, 0, NQ, dev)
    if ones:
        arrays = [np.ones_like(a) for a in arrays]
    _, prog = bench.build_program(cfg)
    return space, arrays, xs, prog


@pytest.mark.parametrize("cfg", CFGS)
def test_partition_of_unity_full_size(cfg):
    space, arrays, xs, prog = _setup(cfg, ones=True)
    ev = Evaluator(space, arrays, prog=prog)
    out = ev(xs)
    out = out[0] if isinstance(out, tuple) else out
    assert float((out - 1).abs().max()) <= 2e-5


@pytest.mark.parametrize("cfg", CFGS)
def test_linearity_full_size(cfg):
    space, arrays, xs, prog = _setup(cfg)
    rng = np.random.default_rng(11)
    other = [rng.random(a.shape).astype(np.float32) for a in arrays]
    mix = [(0.25 * a + 0.5 * b).astype(np.float32) for a, b in zip(arrays, other)]
    outs = []
    for data in (arrays, other, mix):
        r = Evaluator(space, data, prog=prog)(xs)
        outs.append((r[0] if isinstance(r, tuple) else r).double())
    lhs = outs[2]
    rhs = 0.25 * outs[0] + 0.5 * outs[1]
    assert float((lhs - rhs).abs().max()) <= 1e-5


@pytest.mark.parametrize("cfg", CFGS)
def test_oracle_spot_check_full_size(cfg):
    space, arrays, xs, prog = _setup(cfg)
    ev = Evaluator(space, arrays, prog=prog)
    r = ev(xs)
    got = (r[0] if isinstance(r, tuple) else r)[:1500].double().cpu().numpy()
    osp = refeval.load_space_file(SPACES_DIR / f"{space.name}.json")
    sample = xs[:1500].double().cpu().numpy()
    grad = prog.has_grad
    ref = refeval.reference_eval_batch(osp, sample, [a.astype(np.float64) for a in arrays], grad=grad)
    want = ref[0] if grad else ref
    assert np.all(np.abs(got - want) <= 1e-6 + 1e-5 * np.maximum(np.abs(got), np.abs(want)))
    if grad:
        g = r[1][:1500].double().cpu().numpy()
        assert np.abs(g - ref[1]).max() <= 1e-5 * max(1.0, float(np.abs(ref[1]).max()))


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_direct_and_binned_agree_full_size(cfg):
    space, arrays, xs, prog = _setup(cfg)
    a = Evaluator(space, arrays, prog=prog)(xs)
    _, p2 = bench.build_program(cfg, mode="direct")
    b = Evaluator(space, arrays, prog=p2)(xs)
    assert torch.equal(a, b) or float((a - b).abs().max()) <= 1e-6


def test_multi_rank_bench_code_path():
    """bench.py under torchrun with 2 ranks (gloo so both ranks can share the one GPU of
    the test box): per-rank shards, volume broadcast, max-over-ranks timing, one line."""
    import json
    import os
    import subprocess
    import sys
    env = dict(os.environ, SPLINEGPU_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
           "--config", "c1", "--steps", "3", "--warmup", "3", "--no-cpu", "--gather"]
    r = subprocess.run(cmd, cwd=str(bench.ROOT), env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["parallelism"].startswith("query shards x2")
    assert d["gather_ms"] is not None and d["gather_ms"] > 0


SELECT_CFGS = ["c1", "c2", "c3", "c4", "c4v", "c4v4", "c5", "c5u", "c3o2"]


@pytest.mark.parametrize("cfg", SELECT_CFGS)
def test_selection_bit_exact_full_size(cfg):
    """The exact bench kernel variant with dbg=True at the configuration's full extents:
    lattice shift k and sub-region of every (query, coset) bit-exact against the oracle on
    >= 64K adversarial queries scaled to those extents (k + 1/2 +- ulp, |x| < 1e-9 at coset
    offsets, on-plane points, out-of-range) plus bin-edge / wrap-border points and a slice
    of the configuration's own query stream; values against the oracle on a subset."""
    from tests.adversarial import adversarial_points, border_points
    c = bench.CONFIGS[cfg]
    dev = torch.device("cuda", 0)
    space, arrays, _ = bench.make_inputs(cfg, 0, dev)
    _, prog = bench.build_program(cfg, dbg=True)
    ev = Evaluator(space, arrays, prog=prog)
    rng = np.random.default_rng(31)
    ext = c["extents"]
    sets = [adversarial_points(space, ext, rng, 1 << 16),
            border_points(ext, prog.bin or prog.presort, rng, 1 << 14),
            bench.make_queries(cfg, 0, 1 << 14, dev).double().cpu().numpy()]
    xs = np.concatenate(sets).astype(np.float32)
    assert len(xs) >= 1 << 16
    osp = refeval.load_space_file(SPACES_DIR / f"{space.name}.json")
    # the fp64 oracle itself raises UnreachableRegionError on a few of these (e.g. a
    # denormal coordinate next to a plane vertex: the rounded dot products give a sign
    # vector no region has, oracle.py:56-74); the kernel must flag exactly those
    x64 = xs.astype(np.float64)
    bad = np.zeros(len(xs), dtype=bool)
    for off in osp.cosets:
        _, xloc = refeval.rho(osp, x64 - np.array([float(q) for q in off]))
        if osp.planes:
            bad |= np.array(osp.sigma, dtype=np.int64)[refeval.plane_q(osp, xloc)] < 0
    if bad.any():
        from paper_2102_08518_b200 import UnreachableRegionError
        with pytest.raises(UnreachableRegionError):
            ev(torch.from_numpy(xs[bad][:1]).cuda())
        xs = xs[~bad]
    r = ev(torch.from_numpy(xs).cuda())
    out, dbg = r[0], r[2]
    dbg = dbg.cpu().numpy()
    x64 = xs.astype(np.float64)
    s = space.dim
    for ci, (k, sub) in enumerate(refeval.selection(osp, x64)):
        bad = np.flatnonzero((dbg[:, ci, :s] != k).any(axis=1) | (dbg[:, ci, s] != sub))
        assert bad.size == 0, (cfg, ci, bad[:5], x64[bad[:5]])
    pick = rng.choice(len(xs), size=3000, replace=False)
    grad = prog.has_grad
    ref = refeval.reference_eval_batch(osp, x64[pick], [a.astype(np.float64) for a in arrays],
                                       grad=grad)
    want = ref[0] if grad else ref
    got = out.double().cpu().numpy()[pick]
    assert np.all(np.abs(got - want) <= 1e-6 + 1e-5 * np.maximum(np.abs(got), np.abs(want)))
