"""Build libsplinegpu.so (the C-ABI boundary) in-tree with nvcc for sm_100a."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = CUDA / "bin" / "nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def build_library(force: bool = False, verbose: bool = False) -> Path:
    src = PKG / "csrc" / "sg_api.cu"
    hdr = PKG.parent / "include" / "splinegpu.h"
    out = PKG / "libsplinegpu.so"
    if (not force and out.exists()
            and out.stat().st_mtime > max(src.stat().st_mtime, hdr.stat().st_mtime)):
        return out
    cmd = [str(NVCC), "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", *ARCH, "-lineinfo",
           "-cudart", "static", "-o", str(out), str(src), f"-L{CUDA / 'lib64'}", "-lnvrtc",
           "-Xlinker", f"-rpath,{CUDA / 'lib64'}"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return out


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
