"""One small launch per execution mode, for compute-sanitizer (run under gpurun):

    compute-sanitizer --tool memcheck  python tools/sanitize.py direct
    compute-sanitizer --tool racecheck python tools/sanitize.py sorted

Modes: direct, binned (TMA bricks + the query sort kernels), sorted (psi-sorted persistent
tiles, class-major warp chunks), sorted_table (dynamic-smem coefficient tables, site loop,
two pairs per thread), presort_grad (locality presort + gradient, c4v's shape), render
(sorted ray blocks).  Each launch is checked against the
oracle so a sanitizer run also proves the launch did its work.
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import refeval  # noqa: E402
from paper_2102_08518_b200 import Evaluator, GenConfig, ScheduleParams  # noqa: E402
from tests.gpu_util import close, load_golden  # noqa: E402

MODES = {
    "direct": ("bcc_voronoi2", dict(mode="direct")),
    "binned": ("bcc_box5", dict(mode="binned", form="sym")),
    "sorted": ("bcc_voronoi3", dict(mode="sorted", radix=1, block=640, tile=3200, cmajor=3,
                                    min_blocks=1)),
    "sorted_table": ("bcc_voronoi3", dict(mode="sorted", radix=1, coeffs="table", tloop=1,
                                          tpairs=2, block=256)),
    # c4v's shape: locality presort (sort kernels) + sym form + gradient, affine offsets
    "presort_grad": ("fcc_voronoi3", dict(mode="sorted", form="sym", radix=1, presort=1, grad=True,
                                          block=640, tile=1280, min_blocks=1)),
}


def main(mode):
    if mode == "render":
        from paper_2102_08518_b200.render import Renderer
        space, ospace, z, arrays = load_golden("bcc_voronoi3")
        r = Renderer(space, arrays, 16, 8, 40)
        img = r()
        torch.cuda.synchronize()
        assert torch.isfinite(img).all()
        print("render ok", tuple(img.shape))
        return
    name, kw = MODES[mode]
    space, ospace, z, arrays = load_golden(name)
    cfg = GenConfig(ScheduleParams(1, space.stencil_size), float_width="f32", dbg=True, **kw)
    ev = Evaluator(space, arrays, cfg)
    xs = np.concatenate([z["uniform_xs"], z["adversarial_xs"]]).astype(np.float32)
    out, _, dbg = ev(torch.from_numpy(xs).cuda())
    got = out.double().cpu().numpy()
    want = refeval.reference_eval_batch(ospace, xs.astype(np.float64),
                                        [a.astype(np.float64) for a in arrays])
    assert close(got, want, 1e-5, 1e-6).all()
    print(f"{mode} ok: {name}, {len(xs)} queries, max err {np.abs(got - want).max():.2e}")


if __name__ == "__main__":
    main(sys.argv[1])
