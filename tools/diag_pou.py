"""Partition-of-unity diagnostic over kernel variants of one bench configuration (all-ones
volume -> every query must give 1): python tools/diag_pou.py c4v [n]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_08518_b200 import Evaluator  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4v"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
c = bench.CONFIGS[cfg]
dev = torch.device("cuda", 0)
space, arrays, xs = bench.make_inputs(cfg, 0, dev)
xs = xs[:n].contiguous()
ones = [np.ones_like(a) for a in arrays]
VARS = {
    "bench": {},
    "presort0": dict(presort=0),
    "horner": dict(form="horner"),
    "horner_presort0": dict(form="horner", presort=0),
    "nograd": dict(grad=False),
    "direct_table": dict(mode="direct", coeffs="table", presort=0, form="horner", block=128),
    "tc": dict(form="horner", coeffs="table", tc=1, block=384, presort=0, cmajor=0),
}
for name, over in VARS.items():
    try:
        over = dict(over)
        g = over.pop("grad", c["grad"])
        from paper_2102_08518_b200 import generate, load_fixture
        sp = load_fixture(c["space"])
        kw = dict(c.get("variant", {}))
        kw.update(over)
        prog = generate(sp, bench.gen_config_for(sp, g, **kw), c["extents"])
        ev = Evaluator(space, ones, prog=prog)
        out = ev(xs)
        out = out[0] if isinstance(out, tuple) else out
        torch.cuda.synchronize()
        err = (out - 1).abs()
        bad = int((err > 2e-5).sum())
        print(f"{cfg} {name:18s} max|f-1| = {float(err.max()):.3e}  bad {bad}/{n}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{cfg} {name:18s} FAILED {type(e).__name__}: {str(e)[:200]}", flush=True)
