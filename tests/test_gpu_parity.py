"""CUDA path vs the oracle / the reference's golden vectors (needs a B200).

Bar (north_star): lattice shift k and sub-region index bit-exact for every
query and coset; values within 1e-5 relative (f32 kernels vs the fp64
reference) and 1e-12 for the f64 variant.  Every test goes through the C ABI
(libsplinegpu.so) with an NVRTC-compiled sm_100a kernel.
"""

import itertools

import numpy as np
import pytest

from oracle import refeval
from tests.gpu_util import (ATOL_F32, ATOL_F64, RTOL_F32, RTOL_F64, close, golden_names,
                            load_golden)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SETS = ("uniform", "grid", "adversarial")


def _evaluator(space, arrays, **kw):
    from paper_2102_08518_b200 import Evaluator, GenConfig, ScheduleParams
    n = space.stencil_size
    params = kw.pop("params", ScheduleParams(1, n, "predicated"))
    fw = kw.pop("float_width", "f32")
    if kw.get("pack") == 2 and not space.uniform_stencils:
        pytest.skip("pack=2 needs one stencil size for every sub-region")
    dt = np.float32 if fw == "f32" else np.float64
    cfg = GenConfig(params=params, float_width=fw, **kw)
    try:
        return Evaluator(space, [a.astype(dt) for a in arrays], cfg)
    except ValueError as e:
        if "48 KB static limit" in str(e):
            pytest.skip(str(e))
        raise


def _xs(z, which, dtype=torch.float32):
    return torch.from_numpy(z[f"{which}_xs"].astype(np.float64)).to(dtype).cuda()


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("mode", ["direct", "binned", "sorted", "direct_f64", "pack2", "pack2_binned",
                                  "radix", "radix_f64", "presort"])
def test_selection_bit_exact(name, mode):
    space, _, z, arrays = load_golden(name)
    if _big(space) and mode not in ("sorted", "radix", "radix_f64", "presort"):
        pytest.skip("variant not meant for order-4 spaces")
    if mode == "direct_f64":
        ev = _evaluator(space, arrays, dbg=True, select="f64")
    elif mode == "presort":
        ev = _evaluator(space, arrays, dbg=True, mode="sorted", presort=4)
    elif mode.startswith("radix"):
        ev = _evaluator(space, arrays, dbg=True, radix=1, mode="sorted",
                        select="f64" if mode.endswith("f64") else "auto")
    elif mode.startswith("pack2"):
        ev = _evaluator(space, arrays, dbg=True, pack=2,
                        mode="binned" if mode.endswith("binned") else "direct")
    else:
        ev = _evaluator(space, arrays, dbg=True, mode=mode)
    for which in SETS:
        out, _, dbg = ev(_xs(z, which))
        dbg = dbg.cpu().numpy()
        k_want, sub_want = z[f"{which}_k"], z[f"{which}_sub"]
        s = space.dim
        for ci in range(space.ncosets):
            assert np.array_equal(dbg[:, ci, :s], k_want[ci]), (which, ci)
            assert np.array_equal(dbg[:, ci, s], sub_want[ci]), (which, ci)


CONFIGS = [
    dict(),
    dict(form="sites"),
    dict(coeffs="lut"),
    dict(unroll_cosets=False),
    dict(params_mode="branchy"),
    dict(params_mode="branchy", form="sites"),
    dict(params_md=(2, 4)),
    dict(params_md=(2, 4), refetch=True),
    dict(block=256),
    dict(mode="binned"),
    dict(mode="binned", stage="ldg", unroll_cosets=False),
    dict(mode="binned", form="sites", block=256),
    dict(coeffs="table"),
    dict(coeffs="table", mode="binned", params_md=(2, 4)),
    dict(form="sym"),
    dict(form="sym", mode="binned", params_mode="branchy"),
    dict(mode="sorted"),
    dict(select="f64"),
    dict(pack=2),
    dict(radix=1),
    dict(radix=1, mode="sorted", select="f64"),
    dict(mode="sorted", rank="atomic", radix=1),
    dict(mode="sorted", presort=4, radix=1),
    dict(mode="sorted", presort=8, form="sym", tile=512, block=256),
    dict(pack=2, mode="binned", form="sym"),
    dict(pack=2, form="sites", params_md=(2, 4)),
    dict(pack=2, mode="binned", block=256, select="f64"),
    dict(select="f64", mode="binned"),
    dict(select="f64", mode="sorted", form="sym"),
    dict(mode="sorted", form="sym", block=256, tile=512),
    dict(mode="sorted", coeffs="table", tile=256),
    dict(mode="sorted", params_md=(2, 4), form="sites"),
    dict(mode="sorted", coeffs="table", tloop=1),
    dict(mode="sorted", coeffs="table", tloop=1, tpairs=2, block=256, radix=1),
    dict(coeffs="table", tloop=1),
    dict(mode="sorted", radix=1, fetch_offsets="table"),
    dict(mode="sorted", radix=1, gtables="sg_Tq,sg_aff0,sg_off0,sg_psi,sg_sigma"),
    dict(mode="sorted", radix=1, cmajor=3, cflip=1, tile=256, block=128),
    dict(mode="sorted", radix=1, qhoist=1, tile=512, block=128),
    dict(mode="sorted", radix=1, qhoist=1, presort=4, tile=512, block=128),
]


def _cfg(space, spec):
    from paper_2102_08518_b200 import ScheduleParams
    spec = dict(spec)
    n = space.stencil_size
    m, d = spec.pop("params_md", (1, n))
    m, d = min(m, n), min(max(d, min(m, n)), n)
    mode = spec.pop("params_mode", "predicated")
    refetch = spec.pop("refetch", False)
    spec["params"] = ScheduleParams(m, d, mode, refetch)
    return spec


def _big(space):
    """Order-4 spaces (thousands of terms per polynomial): only the variants meant for them
    (sorted dispatch, branchy arms, table site loop) -- predicated immediates of 4 x 3,000
    terms compile for minutes and spill."""
    return max(len(rp.poly.terms) for rp in space.ref_polys) > 1500


def _big_ok(spec):
    return spec.get("mode") == "sorted" or spec.get("tloop") or spec.get("params_mode") == "branchy"


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("ci", range(len(CONFIGS)))
def test_values_f32_vs_reference(name, ci):
    space, _, z, arrays = load_golden(name)
    if _big(space) and not _big_ok(CONFIGS[ci]):
        pytest.skip("variant not meant for order-4 spaces")
    ev = _evaluator(space, arrays, **_cfg(space, CONFIGS[ci]))
    for which in SETS:
        got = ev(_xs(z, which)).double().cpu().numpy()
        want = z[f"{which}_value"]
        ok = close(got, want, RTOL_F32, ATOL_F32)
        assert ok.all(), (which, float(np.abs(got - want).max()))


@pytest.mark.parametrize("name", golden_names())
def test_values_f64_variant(name):
    space, _, z, arrays = load_golden(name)
    if _big(space):
        pytest.skip("f64 predicated immediates of order-4 spaces: see _big")
    for spec in (dict(), dict(params_mode="branchy", form="sites"), dict(unroll_cosets=False)):
        ev = _evaluator(space, arrays, float_width="f64", **_cfg(space, spec))
        for which in SETS:
            got = ev(_xs(z, which, torch.float64)).cpu().numpy()
            want = z[f"{which}_value"]
            ok = close(got, want, RTOL_F64, ATOL_F64)
            assert ok.all(), (which, spec, float(np.abs(got - want).max()))


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("mode", ["direct", "binned", "table", "sym", "sorted", "sorted_sym",
                                  "pack2", "pack2_binned_sym", "presort", "sorted_table_pairs",
                                  "table_loop"])
def test_gradient_vs_oracle(name, mode):
    space, ospace, z, arrays = load_golden(name)
    if _big(space) and mode not in ("sorted_table_pairs", "table_loop"):
        pytest.skip("variant not meant for order-4 spaces")
    xs = z["uniform_xs"].astype(np.float64)
    _, gwant = refeval.reference_eval_batch(ospace, xs, [a.astype(np.float64) for a in arrays],
                                            grad=True)
    if mode == "table":
        ev = _evaluator(space, arrays, grad=True, coeffs="table")
    elif mode == "sym":
        ev = _evaluator(space, arrays, grad=True, form="sym")
    elif mode == "sorted_sym":
        ev = _evaluator(space, arrays, grad=True, form="sym", mode="sorted", block=256)
    elif mode == "pack2":
        ev = _evaluator(space, arrays, grad=True, pack=2)
    elif mode == "presort":
        ev = _evaluator(space, arrays, grad=True, mode="sorted", presort=4)
    elif mode == "table_loop":
        ev = _evaluator(space, arrays, grad=True, mode="sorted", coeffs="table", tloop=1, block=256)
    elif mode == "sorted_table_pairs":
        if _big(space):
            pytest.skip("two pairs per thread need one monomial pass")
        ev = _evaluator(space, arrays, grad=True, mode="sorted", coeffs="table", tloop=1, tpairs=2,
                        block=256)
    elif mode == "pack2_binned_sym":
        ev = _evaluator(space, arrays, grad=True, pack=2, mode="binned", form="sym")
    else:
        ev = _evaluator(space, arrays, grad=True, mode=mode)
    out, g, _ = ev(_xs(z, "uniform"))
    g = g.double().cpu().numpy()
    scale = max(1.0, float(np.abs(gwant).max()))
    assert np.abs(g - gwant).max() <= 1e-5 * scale


@pytest.mark.parametrize("name", golden_names())
@pytest.mark.parametrize("mode", ["direct", "binned", "sorted", "pack2", "presort"])
def test_host_path_matches_device_path(name, mode):
    space, _, z, arrays = load_golden(name)
    if _big(space) and mode != "sorted":
        pytest.skip("variant not meant for order-4 spaces")
    if mode == "pack2":
        ev = _evaluator(space, arrays, pack=2)
    elif mode == "presort":
        ev = _evaluator(space, arrays, mode="sorted", presort=4)
    else:
        ev = _evaluator(space, arrays, mode=mode)
    xs = z["uniform_xs"]
    dev = ev(torch.from_numpy(xs).cuda()).cpu().numpy()
    host = ev.eval_host(xs, chunk=257)
    assert np.array_equal(dev, host)


def test_unreachable_sigma_raises():
    """sigma == -1 -> UnreachableRegionError (reference ir.py:757-766, oracle.py:69-73)."""
    import dataclasses
    from paper_2102_08518_b200 import Evaluator, GenConfig, ScheduleParams, UnreachableRegionError
    from paper_2102_08518_b200.cudagen import generate
    from paper_2102_08518_b200.model import SubRegionIndexer
    space, _, z, arrays = load_golden("zp")
    sig = list(space.indexer.sigma)
    sig[0] = -1   # q == 0: x0 - x1 < 0 and x0 + x1 < 0
    bad = dataclasses.replace(space, indexer=SubRegionIndexer(4, tuple(sig)))
    prog = generate(bad, GenConfig(ScheduleParams(1, 7)), (8, 8), validate=False)
    ev = Evaluator(bad, arrays, prog=prog)
    ev(torch.tensor([[0.1, 0.3]], dtype=torch.float32).cuda())          # q = 2: fine
    with pytest.raises(UnreachableRegionError):
        ev(torch.tensor([[-0.3, 0.1]], dtype=torch.float32).cuda())     # q = 0
    ev(torch.tensor([[0.1, 0.3]], dtype=torch.float32).cuda())          # flag was cleared


def test_reference_contract_interpret_batch():
    """interpret_batch keeps the reference signature: numpy in, numpy (N,) out."""
    from paper_2102_08518_b200 import DataVolume, GenConfig, ScheduleParams, generate, interpret_batch
    space, _, z, arrays = load_golden("trilinear_voronoi")
    data = DataVolume(arrays)
    prog = generate(space, GenConfig(ScheduleParams(2, 5, "branchy")), (6, 6, 6))
    xs = z["uniform_xs"].astype(np.float64)
    got = interpret_batch(prog, xs, data)
    assert got.shape == (xs.shape[0],) and got.dtype == np.float64
    assert close(got, z["uniform_value"], RTOL_F32, ATOL_F32).all()


def test_binned_module_on_two_streams():
    """One binned module (one sort scratch) used from two streams at once: the library
    orders the launches, so both results equal the single-stream ones."""
    from paper_2102_08518_b200 import runtime
    space, _, z, arrays = load_golden("bcc_box5")
    ev = _evaluator(space, arrays, mode="binned")
    rng = np.random.default_rng(5)
    E = np.array(arrays[0].shape, np.float32)
    xa = torch.from_numpy((rng.random((300000, 3)) * E).astype(np.float32)).cuda()
    xb = torch.from_numpy((rng.random((200000, 3)) * E).astype(np.float32)).cuda()
    want_a, want_b = ev(xa).clone(), ev(xb).clone()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    oa = torch.empty(xa.shape[0], device="cuda")
    ob = torch.empty(xb.shape[0], device="cuda")
    torch.cuda.synchronize()
    for _ in range(5):
        runtime.eval_device(ev.module, ev.volume, xa, oa, stream=sa)
        runtime.eval_device(ev.module, ev.volume, xb, ob, stream=sb)
    torch.cuda.synchronize()
    assert torch.equal(oa, want_a) and torch.equal(ob, want_b)


@pytest.mark.parametrize("mode", ["direct", "binned", "sorted"])
def test_empty_and_tiny_batches(mode):
    """n = 0 is a no-op; n = 1 and n = 33 (ragged tiles / warps) match the oracle."""
    space, ospace, z, arrays = load_golden("bcc_voronoi2")
    ev = _evaluator(space, arrays, mode=mode)
    out = ev(torch.zeros((0, 3), dtype=torch.float32, device="cuda"))
    assert out.shape == (0,)
    for n in (1, 33):
        xs = z["uniform_xs"][:n].astype(np.float32)
        got = ev(torch.from_numpy(xs).cuda()).double().cpu().numpy()
        want = refeval.reference_eval_batch(ospace, xs.astype(np.float64),
                                            [a.astype(np.float64) for a in arrays])
        assert close(got, want, RTOL_F32, ATOL_F32).all()
    host = ev.eval_host(z["uniform_xs"][:0].astype(np.float32))
    assert host.shape == (0,)


def test_sorted_host_path_repeats_bit_exact():
    """The persistent sorted kernel claims tiles from a per-launch counter slot: the
    pipelined host path (3 streams, chunks of 257 queries -> thousands of overlapping
    launches of one module) equals the device path bit for bit, every time."""
    space, _, z, arrays = load_golden("bcc_voronoi2")
    ev = _evaluator(space, arrays, mode="sorted", radix=1)
    rng = np.random.default_rng(21)
    E = np.array(arrays[0].shape, np.float32)
    xs = (rng.random((1 << 20, 3)) * E).astype(np.float32)
    dev = ev(torch.from_numpy(xs).cuda()).cpu().numpy()
    for _ in range(50):
        assert np.array_equal(ev.eval_host(xs, chunk=257), dev)


@pytest.mark.parametrize("kind", ["sorted", "render"])
def test_persistent_modules_on_two_streams(kind):
    """Sorted and sorted-render modules launched concurrently from two streams (their
    tile / ray-block counters must not be shared between launches)."""
    from paper_2102_08518_b200 import runtime
    name = "bcc_voronoi3" if "bcc_voronoi3" in golden_names() else "bcc_voronoi2"
    space, _, z, arrays = load_golden(name)
    rng = np.random.default_rng(22)
    E = np.array(arrays[0].shape, np.float32)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    if kind == "sorted":
        ev = _evaluator(space, arrays, mode="sorted", radix=1)
        xa = torch.from_numpy((rng.random((400000, 3)) * E).astype(np.float32)).cuda()
        xb = torch.from_numpy((rng.random((300001, 3)) * E).astype(np.float32)).cuda()
        want_a, want_b = ev(xa).clone(), ev(xb).clone()
        oa = torch.empty(xa.shape[0], device="cuda")
        ob = torch.empty(xb.shape[0], device="cuda")
        torch.cuda.synchronize()
        for _ in range(8):
            runtime.eval_device(ev.module, ev.volume, xa, oa, stream=sa)
            runtime.eval_device(ev.module, ev.volume, xb, ob, stream=sb)
            torch.cuda.synchronize()
            assert torch.equal(oa, want_a) and torch.equal(ob, want_b)
            oa.zero_(), ob.zero_()
        return
    from paper_2102_08518_b200.render import Renderer
    from paper_2102_08518_b200.queries import ray_table
    r = Renderer(space, arrays, 96, 64, 96)
    rays_b = torch.from_numpy(ray_table(tuple(int(e) for e in E), 64, 48, 160, 5)).cuda()
    rgba_b = torch.empty((64 * 48, 4), dtype=torch.float32, device="cuda")

    def launch_b(stream=None):
        runtime.render_device(r.ev.module, r.ev.volume, rays_b, 160, r.tf, rgba_b, stream)
    want_a = r.launch().clone()
    launch_b()
    want_b = rgba_b.clone()
    torch.cuda.synchronize()
    for _ in range(8):
        r.rgba.zero_(), rgba_b.zero_()
        torch.cuda.synchronize()
        r.launch(sa)
        launch_b(sb)
        torch.cuda.synchronize()
        assert torch.equal(r.rgba, want_a) and torch.equal(rgba_b, want_b)


def test_volume_replicate():
    """sg_volume_replicate: the replica (same GPU here; a peer copy over NVLink across GPUs
    when more than one is visible) evaluates bit-identically to the original."""
    from paper_2102_08518_b200 import runtime
    space, _, z, arrays = load_golden("bcc_voronoi3" if "bcc_voronoi3" in golden_names() else "bcc_box5")
    ev = _evaluator(space, arrays, mode="sorted", radix=1)
    xs = torch.from_numpy(z["uniform_xs"]).cuda()
    want = ev(xs)
    devs = list(range(torch.cuda.device_count()))
    for dev in devs[:2]:
        rep = ev.volume.replicate(dev)
        assert rep.nbytes == ev.volume.nbytes
        if dev == ev.device:
            out = torch.empty_like(want)
            runtime.eval_device(ev.module, rep, xs, out)
            torch.cuda.synchronize()
            assert torch.equal(out, want)
        else:
            from paper_2102_08518_b200.runtime import Module
            mod = Module(ev.prog, dev)
            with torch.cuda.device(dev):
                x2 = xs.to(f"cuda:{dev}")
                out = torch.empty(x2.shape[0], device=f"cuda:{dev}")
                runtime.eval_device(mod, rep, x2, out)
                torch.cuda.synchronize(dev)
            assert torch.equal(out.cpu(), want.cpu())
