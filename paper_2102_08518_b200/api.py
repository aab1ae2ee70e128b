"""Reference-facing Python API (drop-in for the hot path of `splinegen`).

Mirrors the reference's public surface for the evaluation path
(pkg/src/splinegen/__init__.py:10-48):

  generate(space, GenConfig) -> Program             (codegen.py:508; extent-free,
                                                     specialized per volume on use)
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


class Program:
    """The result of the reference-shaped call `generate(space, cfg)` (codegen.py:508): a
    program that does not yet know the volume it will run on.

    The CUDA kernel is specialized on the padded per-coset strides (every stencil fetch
    offset becomes an immediate), so the concrete `CudaProgram` is generated on first use
    for each distinct set of data extents (`specialize`) -- `interpret_batch` and
    `Evaluator` do that transparently, which is what lets the reference's
    `prog = generate(space, cfg); interpret_batch(prog, xs, data)` pattern run unchanged
    for any DataVolume."""

    def __init__(self, space, config: GenConfig | None = None):
        if not isinstance(space, SplineSpace):
            space = SplineSpace.adopt(space)
        self.space = space
        self.config = config or default_config(space)
        self._specs = {}
        # validate the space and the variant once, up front (the reference's generate
        # raises here too), on a nominal geometry
        self.specialize((64,) * space.dim)

    name = property(lambda self: self.space.name)
    dim = property(lambda self: self.space.dim)
    ncosets = property(lambda self: self.space.ncosets)
    float_width = property(lambda self: self.config.float_width)

    @property
    def dtype(self):
        return np.float32 if self.config.float_width == "f32" else np.float64

    def specialize(self, extents) -> CudaProgram:
        ext = tuple(tuple(int(v) for v in e) for e in extents) \
            if isinstance(extents[0], (tuple, list)) else tuple(int(v) for v in extents)
        prog = self._specs.get(ext)
        if prog is None:
            prog = self._specs[ext] = _generate(self.space, self.config, ext)
        return prog


def generate(space, config: GenConfig | None = None, extents=None):
    """Reference `generate(space, GenConfig)` (codegen.py:508).

    Without `extents` the result is an extent-free `Program` (specialized per volume on
    first use); with `extents` (one tuple of s ints, or one per coset) the concrete
    `CudaProgram` for that geometry is returned directly."""
    if extents is None:
        return Program(space, config)
    return _generate(space, config, extents)


def _specialize_for(prog, arrays):
    ext = tuple(tuple(int(e) for e in a.shape) for a in arrays)
    return prog.specialize(ext if len(set(ext)) > 1 else ext[0])


class Evaluator:
    """A generated kernel bound to a device-resident volume.

    >>> ev = Evaluator(space, data, GenConfig(...))      # compile + upload once
    >>> out = ev(xs_tensor)                              # torch (N, s) cuda -> (N,) cuda
    """

    def __init__(self, space, data, config: GenConfig | None = None, device: int = 0,
                 prog=None, module=None):
        import torch
        if not isinstance(space, SplineSpace):
            space = SplineSpace.adopt(space)
        self.space = space
        arrays = data.arrays if hasattr(data, "arrays") else list(data)
        if len(arrays) != space.ncosets:
            raise InterpreterError(f"data has {len(arrays)} cosets, program wants {space.ncosets}")
        ext = tuple(tuple(int(e) for e in a.shape) for a in arrays)
        if isinstance(prog, Program):
            prog = _specialize_for(prog, arrays)
        self.prog = prog or _generate(space, config or default_config(space), ext)
        if self.prog.extents != ext:
            raise InterpreterError(f"program compiled for extents {self.prog.extents}, data has {ext}")
        self.device = device
        self.module = module if module is not None else runtime.Module(self.prog, device)
        self.volume = runtime.Volume(arrays, self.prog.halo, self.prog.dtype, device,
                                     padded=self.prog.padded_extents)
        self.torch_dtype = torch.float32 if self.prog.float_width == "f32" else torch.float64

    def __call__(self, xs, out=None, grad=None, dbg=None, check=True):
        import torch
        s, M = self.space.dim, self.space.ncosets
        if xs.ndim != 2 or xs.shape[1] != s:
            raise InterpreterError(f"expected points of shape (N, {s})")
        for name, t in (("xs", xs), ("out", out), ("grad", grad), ("dbg", dbg)):
            if t is not None and (not t.is_cuda or t.device.index != self.device):
                raise InterpreterError(f"{name} must be a CUDA tensor on cuda:{self.device}, "
                                       f"not {t.device}")
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


DEFAULT_BUDGET = 50_000_000   # the reference interpreter's instruction budget (ir.py)

_MODULES = {}   # CudaProgram source key -> loaded module (compiled kernels are reused)


def _module_for(cprog, device=0):
    key = (cprog.key, device)
    mod = _MODULES.get(key)
    if mod is None:
        if len(_MODULES) >= 32:
            _MODULES.clear()
        mod = _MODULES[key] = runtime.Module(cprog, device)
    return mod


def interpret_batch(prog, xs, data, max_steps: int = DEFAULT_BUDGET, counter=None) -> np.ndarray:
    """Reference-contract batch evaluation on the GPU (ir.py:582-700).

    `prog`: a `Program` / `CudaProgram` from `generate`, or a SplineSpace (the default
    config is generated for it).  Like the reference, every call reads `data` afresh
    (the volume is uploaded per call, so in-place edits of the arrays are seen; the
    compiled kernel is cached) and returns an array of the program's dtype.

    `counter` (the reference's per-IR-opcode dynamic instruction count) has no meaning
    for a compiled GPU kernel and is rejected explicitly; `max_steps` (the interpreter's
    runaway-loop budget) is validated and otherwise moot -- generated kernels are
    straight-line per query and always terminate."""
    import torch
    if counter is not None:
        raise InterpreterError("counter= counts reference IR instructions; the CUDA program "
                               "has none (use bench.py's F_alg / ncu instruction counts)")
    if not isinstance(max_steps, (int, np.integer)) or max_steps < 1:
        raise InterpreterError(f"max_steps must be a positive integer, not {max_steps!r}")
    if not isinstance(prog, (Program, CudaProgram)):
        prog = Program(prog)
    space = prog.space
    xs = np.asarray(xs, dtype=np.float64)
    if xs.ndim != 2 or xs.shape[1] != space.dim:
        raise InterpreterError(f"expected points of shape (N, {space.dim})")
    if data.ncosets != space.ncosets:
        raise InterpreterError(f"data has {data.ncosets} cosets, program wants {space.ncosets}")
    arrays = data.arrays if hasattr(data, "arrays") else list(data)
    cprog = _specialize_for(prog, arrays) if isinstance(prog, Program) else prog
    ev = Evaluator(space, arrays, prog=cprog, module=_module_for(cprog))
    t = torch.from_numpy(xs.astype(cprog.dtype)).cuda(ev.device)
    res = ev(t)
    if isinstance(res, tuple):
        res = res[0]
    return res.cpu().numpy().astype(cprog.dtype, copy=False)


def interpret(prog, x, data) -> float:
    return float(interpret_batch(prog, np.asarray([list(x)], dtype=np.float64), data)[0])
