"""The C-ABI library loads without a GPU and exports every symbol the header declares."""

import re
from pathlib import Path

from paper_2102_08518_b200 import runtime

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "splinegpu.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(sg_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("sg_compile", "sg_module_load", "sg_volume_create", "sg_eval", "sg_eval_host",
              "sg_module_status", "sg_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = runtime.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(runtime.EXPORTS)


def test_version_and_error_string():
    lib = runtime.lib()
    assert lib.sg_version() >= 100
    assert isinstance(lib.sg_last_error(), bytes)


def test_invalid_arguments_fail_without_gpu():
    import ctypes
    lib = runtime.lib()
    h = ctypes.c_void_p()
    rc = lib.sg_volume_create(0, 9, 1, None, 0, None, 0, None, 0, None, ctypes.byref(h))
    assert rc == runtime.SG_EINVAL
    rc = lib.sg_eval(None, None, None, 0, None, None, None, None)
    assert rc == runtime.SG_EINVAL
    rc = lib.sg_render(None, None, None, 0, 0, None, None, None)
    assert rc == runtime.SG_EINVAL


def test_nvrtc_compiles_for_sm100a_without_gpu():
    src = 'extern "C" __global__ void k(float* p) { p[threadIdx.x] *= 2.0f; }\n'
    img, key = runtime.compile_source(src, use_cache=False)
    assert img[:4] == b"\x7fELF"
