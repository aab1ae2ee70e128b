"""B200-native (sm_100a) evaluator for shift-invariant spline reconstruction.

Drop-in for the hot path of the reference `splinegen` package (arXiv 2102.08518,
Part II): evaluation of  f(x) = sum_cosets sum_j c[l][k + pi_j] psi(T(x - l - k) + t')
for large query batches.  The host keeps the reference's Part-I description and
Python API; `cudagen` lowers it to one-query-per-thread sm_100a kernels that are
compiled with NVRTC and called through the C ABI in include/splinegpu.h.
"""

from .api import DataVolume, Evaluator, InterpreterError, Program, generate, interpret, interpret_batch, make_volume, sample_points
from .cudagen import CudaProgram, GenConfig, default_config
from .model import (
    SplineSpace,
    list_fixtures,
    load_fixture,
    load_space,
    parse_space,
    serialize_space,
    validate_space,
)
from .poly import Poly, group_polynomial, horner_factorize, poly_eval
from .runtime import SplineGpuError, UnreachableRegionError
from .schedule import EvalPlan, ScheduleParams, schedule_pipeline

__all__ = [
    "CudaProgram", "DataVolume", "EvalPlan", "Evaluator", "GenConfig", "InterpreterError", "Poly", "Program",
    "ScheduleParams", "SplineGpuError", "SplineSpace", "UnreachableRegionError", "default_config",
    "generate", "group_polynomial", "horner_factorize", "interpret", "interpret_batch",
    "list_fixtures", "load_fixture", "load_space", "make_volume", "parse_space", "poly_eval",
    "sample_points", "schedule_pipeline", "serialize_space", "validate_space",
]

__version__ = "0.1.0"
