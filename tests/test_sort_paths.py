"""The C ABI's query sort takes different kernels by bin count: the tiled scatter (tile-local
counting sort, coalesced record runs) up to SPLINEGPU_TILED_MAX_BINS bins, the plain scatter
above.  Both must give the oracle's values; the environment knob is read once per process,
so each path runs in its own subprocess (needs a B200)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from oracle import refeval
from paper_2102_08518_b200 import Evaluator, GenConfig, ScheduleParams, load_fixture
from paper_2102_08518_b200.model import SPACES_DIR
space = load_fixture("fcc_voronoi3")
ext = (20, 20, 20)
rng = np.random.default_rng(5)
arrays = [rng.random(ext).astype(np.float32) for _ in range(space.ncosets)]
cfg = GenConfig(ScheduleParams(1, space.stencil_size), mode="sorted", form="sym", radix=1,
                presort=1, block=256)            # 20^3 = 8,000 one-cell bins
ev = Evaluator(space, arrays, cfg)
xs = (rng.random((1 << 16, 3)) * 20).astype(np.float32)
got = ev(torch.from_numpy(xs).cuda()).double().cpu().numpy()
osp = refeval.load_space_file(SPACES_DIR / "fcc_voronoi3.json")
want = refeval.reference_eval_batch(osp, xs[:3000].astype(np.float64), [a.astype(np.float64) for a in arrays])
err = float(np.abs(got[:3000] - want).max())
print(json.dumps({"err": err, "sum": float(got.sum())}))
"""


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], cwd=str(ROOT), env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])


def test_tiled_and_plain_scatter_agree_with_the_oracle():
    plain = _run({})                                          # 8,000 bins > 2,048: plain scatter
    tiled = _run({"SPLINEGPU_TILED_MAX_BINS": "10240"})       # tiled (8,000 x 16 B of bin state + the tile fit)
    assert plain["err"] <= 2e-5 and tiled["err"] <= 2e-5
    assert plain["sum"] == tiled["sum"]
