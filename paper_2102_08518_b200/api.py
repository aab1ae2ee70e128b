"""Reference-facing Python API (drop-in for the hot path of `splinegen`).

Mirrors the reference's public surface for the evaluation path
(pkg/src/splinegen/__init__.py:10-48):

  generate(space, GenConfig) -> CudaProgram         (codegen.py:508)
  interpret_batch(prog, xs, data) -> ndarray (N,)   (ir.py:582-700)
  interpret(prog, x, data) -> float                 (ir.py:793)
  DataVolume(arrays)                                (ir.py:524-558)
  make_volume / sample_points                       (bench.py:57-74)

`interpret_batch` keeps the reference contract (numpy (N, s) in, numpy (N,)
out, DataVolume data, the same ValueError-style shape checks and an
UnreachableRegionError for sigma == -1) but executes the generated sm_100a
kernel.  `Evaluator` is the zero-copy device API for torch tensors.
"""

from __future__ import annotations

import numpy as np

from . import runtime
from .cudagen import CudaProgram, GenConfig, default_config
from .cudagen import generate as _generate
from .model import SplineSpace


class InterpreterError(Exception):
    """Shape / coset mismatch (reference ir.py:591-596)."""


class DataVolume:
    """Per-coset sample arrays with periodic indexing (reference ir.py:524-558)."""

    def __init__(self, arrays):
        arrs = tuple(np.asarray(a) for a in arrays)
        if not arrs:
            raise ValueError("at least one coset array is required")
        dt = arrs[0].dtype
        if dt not in (np.float32, np.float64):
            raise ValueError("sample arrays must be float32 or float64")
        if any(a.dtype != dt for a in arrs):
            raise ValueError("all coset arrays must share a dtype")
        if any(a.ndim != arrs[0].ndim for a in arrs):
            raise ValueError("all coset arrays must share a rank")
        if any(e < 1 for a in arrs for e in a.shape):
            raise ValueError("extents must be positive")
        self.arrays = arrs

    @property
    def ncosets(self):
        return len(self.arrays)

    @property
    def dim(self):
        return self.arrays[0].ndim

    @property
    def extents(self):
        return tuple(a.shape for a in self.arrays)

    def fetch(self, coset, coords):
        arr = self.arrays[coset]
        return arr[tuple(np.asarray(c) % e for c, e in zip(coords, arr.shape))]


def make_volume(space, extents, seed: int, float_width: str = "f64") -> DataVolume:
    """Seeded U[0,1) samples, cosets drawn in order from one generator (bench.py:57-67)."""
    extents = tuple(int(e) for e in extents)
    if len(extents) != space.dim:
        raise ValueError(f"expected {space.dim} extents")
    if any(e < 1 for e in extents):
        raise ValueError("extents must be positive")
    rng = np.random.default_rng(seed)
    dt = np.float64 if float_width == "f64" else np.float32
    return DataVolume([rng.random(extents).astype(dt) for _ in range(space.ncosets)])


def sample_points(space, data, count: int, seed: int) -> np.ndarray:
    """Seeded uniform points in coset 0's periodic box (bench.py:70-74)."""
    rng = np.random.default_rng(seed)
    return rng.random((count, space.dim)) * np.array(data.extents[0], dtype=np.float64)


def generate(space, config: GenConfig | None = None, extents=None) -> CudaProgram:
    """Reference `generate` + the volume extents the kernel is specialized on."""
    return _generate(space, config, extents)


class Evaluator:
    """A generated kernel bound to a device-resident volume.

    >>> ev = Evaluator(space, data, GenConfig(...))      # compile + upload once
    >>> out = ev(xs_tensor)                              # torch (N, s) cuda -> (N,) cuda
    """

    def __init__(self, space, data, config: GenConfig | None = None, device: int = 0,
                 prog: CudaProgram | None = None):
        import torch
        if not isinstance(space, SplineSpace):
            space = SplineSpace.adopt(space)
        self.space = space
        arrays = data.arrays if hasattr(data, "arrays") else list(data)
        if len(arrays) != space.ncosets:
            raise InterpreterError(f"data has {len(arrays)} cosets, program wants {space.ncosets}")
        ext = tuple(tuple(int(e) for e in a.shape) for a in arrays)
        self.prog = prog or _generate(space, config or default_config(space), ext)
        if self.prog.extents != ext:
            raise InterpreterError(f"program compiled for extents {self.prog.extents}, data has {ext}")
        self.device = device
        self.module = runtime.Module(self.prog, device)
        self.volume = runtime.Volume(arrays, self.prog.halo, self.prog.dtype, device,
                                     padded=self.prog.padded_extents)
        self.torch_dtype = torch.float32 if self.prog.float_width == "f32" else torch.float64

    def __call__(self, xs, out=None, grad=None, dbg=None, check=True):
        import torch
        s, M = self.space.dim, self.space.ncosets
        if xs.ndim != 2 or xs.shape[1] != s:
            raise InterpreterError(f"expected points of shape (N, {s})")
        if xs.dtype != self.torch_dtype or not xs.is_contiguous():
            xs = xs.to(self.torch_dtype).contiguous()
        n = xs.shape[0]
        dev = xs.device
        if out is None:
            out = torch.empty(n, dtype=self.torch_dtype, device=dev)
        if self.prog.has_grad and grad is None:
            grad = torch.empty((n, s), dtype=self.torch_dtype, device=dev)
        if self.prog.has_dbg and dbg is None:
            dbg = torch.empty((n, M, s + 1), dtype=torch.int32, device=dev)
        runtime.eval_device(self.module, self.volume, xs, out, grad, dbg)
        if check:
            self.module.status()
        if self.prog.has_grad or self.prog.has_dbg:
            return out, grad, dbg
        return out

    def eval_host(self, xs: np.ndarray, chunk: int = 0):
        """End-to-end host-buffer path (sg_eval_host): numpy in, numpy out."""
        xs = np.ascontiguousarray(xs, dtype=self.prog.dtype)
        out = np.empty(xs.shape[0], dtype=self.prog.dtype)
        grad = np.empty_like(xs) if self.prog.has_grad else None
        runtime.eval_host(self.module, self.volume, xs, out, grad, chunk)
        self.module.status()
        return (out, grad) if grad is not None else out


_EV_CACHE = {}


def interpret_batch(prog, xs, data, max_steps=None, counter=None) -> np.ndarray:
    """Reference-contract batch evaluation on the GPU (ir.py:582-700).

    `prog` may be a CudaProgram (from `generate`) or a SplineSpace (then the
    default GPU config is generated for the data's extents).
    """
    import torch
    if isinstance(prog, CudaProgram):
        space = prog.space
    else:
        space = prog if isinstance(prog, SplineSpace) else SplineSpace.adopt(prog)
        prog = None
    xs = np.asarray(xs, dtype=np.float64)
    if xs.ndim != 2 or xs.shape[1] != space.dim:
        raise InterpreterError(f"expected points of shape (N, {space.dim})")
    if data.ncosets != space.ncosets:
        raise InterpreterError(f"data has {data.ncosets} cosets, program wants {space.ncosets}")
    key = (id(prog) if prog is not None else id(space), id(data))
    ev = _EV_CACHE.get(key)
    if ev is None or ev[1] is not data:
        ev = (Evaluator(space, data, prog=prog), data)
        _EV_CACHE.clear()
        _EV_CACHE[key] = ev
    e = ev[0]
    t = torch.from_numpy(xs.astype(e.prog.dtype)).cuda(e.device)
    res = e(t)
    if isinstance(res, tuple):
        res = res[0]
    return res.double().cpu().numpy()


def interpret(prog, x, data) -> float:
    return float(interpret_batch(prog, np.asarray([list(x)], dtype=np.float64), data)[0])
