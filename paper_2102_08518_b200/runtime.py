"""ctypes binding of libsplinegpu.so (include/splinegpu.h) + cubin cache.

The product path is: `cudagen.generate` -> CUDA source -> NVRTC (sg_compile,
sm_100a) -> cubin cached in-tree -> `sg_module_load` -> `sg_eval` on torch
device tensors.  There is no CPU fallback: if the shared library is missing
or no CUDA device is present, evaluation raises.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import threading
from pathlib import Path

import numpy as np

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libsplinegpu.so"
CACHE_DIR = Path(os.environ.get("SPLINEGPU_CACHE", PKG / "_cache"))
NVRTC_OPTS = ("--gpu-architecture=sm_100a", "-lineinfo", "--std=c++17", "-DNDEBUG",
              "--ptxas-options=-v")

SG_OK, SG_EINVAL, SG_ECUDA, SG_EUNREACHABLE, SG_ECOMPILE, SG_ENOMEM = range(6)
SG_F32, SG_F64 = 0, 1
SG_MAX_COSETS = 8
SG_MAX_DIM = 4


class SplineGpuError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        super().__init__(f"[sg {code}] {msg}")


class UnreachableRegionError(SplineGpuError):
    """A query hit a sigma entry marked -1 (reference ir.py:757-766 / oracle.py:69-73)."""


class sg_module_info(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("ncosets", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("block", ctypes.c_int32), ("has_grad", ctypes.c_int32),
                ("has_dbg", ctypes.c_int32), ("halo", ctypes.c_int32),
                ("queries_per_thread", ctypes.c_int32),
                ("padded_extents", (ctypes.c_int64 * SG_MAX_DIM) * SG_MAX_COSETS),
                ("mode", ctypes.c_int32), ("rounding", ctypes.c_int32),
                ("stage_tma", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("bin", ctypes.c_int32), ("brick", ctypes.c_int32 * SG_MAX_DIM),
                ("extents", ctypes.c_int64 * SG_MAX_DIM), ("chunk", ctypes.c_int32),
                ("static_smem", ctypes.c_int32), ("presort", ctypes.c_int32)]


_lib = None
_lib_lock = threading.Lock()

EXPORTS = {
    "sg_version": ([], ctypes.c_int),
    "sg_last_error": ([], ctypes.c_char_p),
    "sg_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "sg_compile": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p), ctypes.c_int,
                    ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t),
                    ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sg_free": ([ctypes.c_void_p], None),
    "sg_module_load": ([ctypes.c_void_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_int,
                        ctypes.POINTER(sg_module_info), ctypes.POINTER(ctypes.c_void_p)],
                       ctypes.c_int),
    "sg_module_free": ([ctypes.c_void_p], ctypes.c_int),
    "sg_module_regs": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
                        ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "sg_module_status": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32)],
                         ctypes.c_int),
    "sg_volume_create": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                          ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int,
                          ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_void_p,
                          ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
    "sg_volume_free": ([ctypes.c_void_p], ctypes.c_int),
    "sg_volume_bytes": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "sg_volume_coset_ptr": ([ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)],
                            ctypes.c_int),
    "sg_eval": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "sg_eval_host": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64], ctypes.c_int),
    "sg_module_timing": ([ctypes.c_void_p, ctypes.c_int], ctypes.c_int),
    "sg_module_kernel_time": ([ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_int64)], ctypes.c_int),
    "sg_render": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "sg_volume_replicate": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                             ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
}


def lib():
    """Load libsplinegpu.so (build it with `python -m paper_2102_08518_b200.build`)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise SplineGpuError(SG_EINVAL, f"{LIB_PATH} is missing: run __graft_entry__.build()")
            L = ctypes.CDLL(str(LIB_PATH))
            for name, (args, res) in EXPORTS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
    return _lib


def _check(rc):
    if rc != SG_OK:
        msg = lib().sg_last_error().decode(errors="replace")
        if rc == SG_EUNREACHABLE:
            raise UnreachableRegionError(rc, msg)
        raise SplineGpuError(rc, msg)


# -- compilation ------------------------------------------------------------------


def cache_key(source: str, opts=NVRTC_OPTS) -> str:
    h = hashlib.sha256()
    h.update(source.encode())
    h.update("\0".join(opts).encode())
    return h.hexdigest()[:32]


def compile_source(source: str, name="sg_kernel.cu", opts=NVRTC_OPTS, use_cache=True):
    """NVRTC -> cubin bytes (cached in paper_2102_08518_b200/_cache/<key>.cubin)."""
    key = cache_key(source, opts)
    path = CACHE_DIR / f"{key}.cubin"
    if use_cache and path.exists():
        return path.read_bytes(), key
    L = lib()
    arr = (ctypes.c_char_p * len(opts))(*[o.encode() for o in opts])
    img = ctypes.c_void_p()
    n = ctypes.c_size_t()
    log = ctypes.c_void_p()
    rc = L.sg_compile(source.encode(), name.encode(), arr, len(opts), ctypes.byref(img),
                      ctypes.byref(n), ctypes.byref(log))
    log_text = ctypes.string_at(log.value).decode(errors="replace") if log.value else ""
    if log.value:
        L.sg_free(log)
    _check(rc)
    data = ctypes.string_at(img.value, n.value)
    L.sg_free(img)
    CACHE_DIR.mkdir(parents=True, exist_ok=True)
    tmp = path.with_suffix(f".tmp{os.getpid()}")
    tmp.write_bytes(data)
    os.replace(tmp, path)
    (CACHE_DIR / f"{key}.log").write_text(log_text)
    (CACHE_DIR / f"{key}.cu").write_text(source)
    return data, key


def ptxas_info(key: str) -> str:
    p = CACHE_DIR / f"{key}.log"
    return p.read_text() if p.exists() else ""


# -- device objects ----------------------------------------------------------------


def device_count() -> int:
    n = ctypes.c_int()
    rc = lib().sg_device_count(ctypes.byref(n))
    return n.value if rc == SG_OK else 0


class Module:
    """A loaded generated kernel (sg_module)."""

    def __init__(self, prog, device: int = 0):
        self.prog = prog
        self.device = device
        self.image, self.key = compile_source(prog.source, f"{prog.name}.cu")
        info = sg_module_info()
        info.dim = prog.dim
        info.ncosets = prog.ncosets
        info.dtype = SG_F32 if prog.float_width == "f32" else SG_F64
        info.block = prog.block
        info.has_grad = int(prog.has_grad)
        info.has_dbg = int(prog.has_dbg)
        info.halo = prog.halo
        info.queries_per_thread = getattr(prog, "queries_per_thread", 1)
        for c, row in enumerate(prog.padded_extents):
            for d, e in enumerate(row):
                info.padded_extents[c][d] = e
        info.mode = {"binned": 1, "render": 2, "linear": 3}.get(prog.mode, 0)
        info.rounding = prog.rounding
        info.stage_tma = int(prog.stage_tma)
        info.smem_bytes = prog.smem_bytes
        info.bin = prog.bin
        info.chunk = prog.chunk
        for d, e in enumerate(prog.brick):
            info.brick[d] = e
        for d, e in enumerate(prog.extents[0]):
            info.extents[d] = e
        if getattr(prog, "presort", 0):
            info.presort = 1
            info.bin = prog.presort
            info.chunk = 1 << 16        # the sort's work-item list is unused here: keep it short
        h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(self.image, len(self.image))
        _check(lib().sg_module_load(buf, len(self.image), prog.entry.encode(), device,
                                    ctypes.byref(info), ctypes.byref(h)))
        self.handle = h

    def regs(self):
        r, lb = ctypes.c_int(), ctypes.c_int()
        _check(lib().sg_module_regs(self.handle, ctypes.byref(r), ctypes.byref(lb)))
        return r.value, lb.value

    def set_timing(self, enable: bool):
        _check(lib().sg_module_timing(self.handle, int(enable)))

    def kernel_time(self):
        """(summed ms, launches) of the evaluation kernel since the last call."""
        ms, n = ctypes.c_double(), ctypes.c_int64()
        _check(lib().sg_module_kernel_time(self.handle, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def status(self, stream=None):
        f = ctypes.c_uint32()
        _check(lib().sg_module_status(self.handle, _stream_ptr(stream, self.device), ctypes.byref(f)))
        return f.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.sg_module_free(h)
            self.handle = None


class Volume:
    """Coset arrays on the device with a periodic ghost halo (sg_volume)."""

    def __init__(self, arrays, halo: int, dtype, device: int = 0, stream=None, padded=None):
        import torch
        arrs = list(arrays)
        if not arrs:
            raise ValueError("at least one coset array is required")
        if len(arrs) > SG_MAX_COSETS:
            raise ValueError(f"at most {SG_MAX_COSETS} cosets")
        np_dtype = np.dtype(dtype)
        self.dtype = np_dtype
        self.dim = arrs[0].ndim
        self.extents = tuple(tuple(int(e) for e in a.shape) for a in arrs)
        self.halo = halo
        self.device = device
        ext = (ctypes.c_int64 * (len(arrs) * self.dim))(*[e for row in self.extents for e in row])
        on_dev = isinstance(arrs[0], torch.Tensor) and arrs[0].is_cuda
        keep = []
        if on_dev:
            tdt = torch.float32 if np_dtype == np.float32 else torch.float64
            for a in arrs:
                keep.append(a.to(tdt).contiguous())
            ptrs = (ctypes.c_void_p * len(arrs))(*[k.data_ptr() for k in keep])
        else:
            for a in arrs:
                a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
                keep.append(np.ascontiguousarray(a, dtype=np_dtype))
            ptrs = (ctypes.c_void_p * len(arrs))(*[k.ctypes.data for k in keep])
        h = ctypes.c_void_p()
        pad = None
        if padded is not None:
            pad = (ctypes.c_int64 * (len(arrs) * self.dim))(*[e for row in padded for e in row])
        _check(lib().sg_volume_create(device, self.dim, len(arrs), ext, halo, pad,
                                      SG_F32 if np_dtype == np.float32 else SG_F64, ptrs,
                                      int(on_dev), _stream_ptr(stream, device), ctypes.byref(h)))
        self.handle = h
        self.ncosets = len(arrs)

    def replicate(self, device: int, stream=None) -> "Volume":
        """A full copy of this volume (halo included) on `device`: a peer copy over NVLink
        between GPUs, a device-to-device copy on the same GPU (sg_volume_replicate) -- how
        every rank of a multi-GPU run gets its replica without a host round trip."""
        h = ctypes.c_void_p()
        _check(lib().sg_volume_replicate(self.handle, int(device), _stream_ptr(stream, self.device),
                                         ctypes.byref(h)))
        r = Volume.__new__(Volume)
        r.dtype, r.dim, r.extents, r.halo = self.dtype, self.dim, self.extents, self.halo
        r.device, r.ncosets, r.handle = int(device), self.ncosets, h
        return r

    @property
    def nbytes(self):
        b = ctypes.c_int64()
        _check(lib().sg_volume_bytes(self.handle, ctypes.byref(b)))
        return b.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib is not None:
            _lib.sg_volume_free(h)
            self.handle = None


def _stream_ptr(stream, device=None):
    """cudaStream_t of `stream`; None = torch's current stream on `device` (the module's
    device, not whatever device happens to be current)."""
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
        except Exception:  # pragma: no cover
            pass
        return ctypes.c_void_p(0)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def eval_device(module: Module, volume: Volume, xs, out, grad=None, dbg=None, stream=None):
    """Launch on torch device tensors (async on the current torch stream of the module's
    device).  Every tensor must live on that device: a host pointer handed to the kernel
    would fault and poison the CUDA context, so it is rejected here."""
    for name, t in (("xs", xs), ("out", out), ("grad", grad), ("dbg", dbg)):
        if t is not None and (not t.is_cuda or t.device.index != module.device):
            raise SplineGpuError(SG_EINVAL, f"{name} must be a CUDA tensor on cuda:{module.device}, "
                                            f"not {t.device}")
    n = xs.shape[0]
    _check(lib().sg_eval(module.handle, volume.handle, ctypes.c_void_p(xs.data_ptr()), n,
                         ctypes.c_void_p(out.data_ptr()),
                         ctypes.c_void_p(grad.data_ptr() if grad is not None else 0),
                         ctypes.c_void_p(dbg.data_ptr() if dbg is not None else 0),
                         _stream_ptr(stream, module.device)))


def render_device(module: Module, volume: Volume, rays, steps: int, tf, rgba, stream=None):
    """Fused ray-march + reconstruction + compositing (render-mode modules, sg_render)."""
    _check(lib().sg_render(module.handle, volume.handle, ctypes.c_void_p(rays.data_ptr()),
                           rays.shape[0], int(steps), ctypes.c_void_p(tf.data_ptr()),
                           ctypes.c_void_p(rgba.data_ptr()), _stream_ptr(stream, module.device)))


def eval_host(module: Module, volume: Volume, xs: np.ndarray, out: np.ndarray,
              grad: np.ndarray | None = None, chunk: int = 0):
    """End-to-end call with host buffers (pinned recommended)."""
    n = xs.shape[0]
    _check(lib().sg_eval_host(module.handle, volume.handle, ctypes.c_void_p(xs.ctypes.data), n,
                              ctypes.c_void_p(out.ctypes.data),
                              ctypes.c_void_p(grad.ctypes.data if grad is not None else 0), chunk))
