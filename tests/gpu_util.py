"""Shared helpers for the GPU parity tests (not collected: no test_ prefix)."""

from __future__ import annotations

import numpy as np

from oracle import refeval
from tests.conftest import GOLDEN

RTOL_F32 = 1e-5     # north_star: values within 1e-5 relative (fp32 vs the fp64 oracle)
ATOL_F32 = 1e-6     # absolute floor for values near zero (data are U[0,1))
RTOL_F64 = 1e-12    # north_star: 1e-12 for the fp64 variant
ATOL_F64 = 1e-14


def close(got, want, rtol, atol):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return np.abs(got - want) <= atol + rtol * np.maximum(np.abs(got), np.abs(want))


def golden_names():
    return sorted(p.stem for p in (GOLDEN / "spaces").glob("*.json"))


def load_golden(name):
    from paper_2102_08518_b200 import load_space
    space = load_space(GOLDEN / "spaces" / f"{name}.json")
    ospace = refeval.load_space_file(GOLDEN / "spaces" / f"{name}.json")
    z = np.load(GOLDEN / f"{name}.npz")
    arrays = [z[f"vol_{i}"] for i in range(space.ncosets)]
    return space, ospace, z, arrays
