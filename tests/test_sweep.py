"""Sweep harness: reference CSV / matrix formats (CPU) and a small CUDA sweep (GPU)."""

import numpy as np
import pytest

from paper_2102_08518_b200.sweep import (CSV_HEADER, BenchRecord, default_grid, emit_csv,
                                         emit_matrix, parse_csv)


def test_csv_round_trip_and_matrix_shape():
    recs = [BenchRecord("zp", m, d, mode, "cuda", 100, float(m * 10 + d), 0.5)
            for m, d in default_grid(3) for mode in ("predicated", "branchy")]
    text = emit_csv(recs)
    assert text.splitlines()[0] == CSV_HEADER
    assert parse_csv(text) == sorted(recs, key=lambda r: (r.m, r.d, r.branch_mode, r.backend))
    mat = emit_matrix(recs, "predicated").splitlines()
    assert len(mat) == 3 and mat[0].count("\t") == 0 and mat[2].count("\t") == 2


@pytest.mark.gpu
def test_cuda_sweep_zp():
    from paper_2102_08518_b200 import load_space, make_volume
    from paper_2102_08518_b200.sweep import run_sweep
    from tests.conftest import GOLDEN
    sp = load_space(GOLDEN / "spaces" / "zp.json")
    data = make_volume(sp, (64, 64), seed=0, float_width="f32")
    from oracle import refeval
    from paper_2102_08518_b200.model import serialize_space
    osp = refeval.load_space(serialize_space(sp))
    cells = []

    def check(pts, got, cell):
        want = refeval.reference_eval_batch(osp, pts, [np.asarray(a, np.float64) for a in data.arrays])
        tol = cell[-1]
        err = np.abs(got - want)
        assert (err <= 1e-12 + tol * np.maximum(np.abs(got), np.abs(want))).all(), (cell, err.max())
        cells.append(cell[:3])

    recs = run_sweep(sp, data, grid=[(1, 7), (2, 4)], trials=1 << 16, batch_size=1 << 14,
                     check=check)
    assert len(recs) == 4 and all(r.mean_recon_per_sec > 0 for r in recs)
    assert len(cells) == 4
