"""Build libsplinegpu.so (the C-ABI boundary) in-tree with nvcc for sm_100a."""

from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CUDA = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = CUDA / "bin" / "nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _source_hash(src: Path, hdr: Path) -> str:
    h = hashlib.sha256()
    for p in (src, hdr, Path(__file__)):
        h.update(p.read_bytes())
    return h.hexdigest()


def build_library(force: bool = False, verbose: bool = False) -> Path:
    """Rebuild unless the library was built from exactly these sources (content hash in
    libsplinegpu.so.sha256 -- modification times are not trusted: a copied tree can
    carry a stale binary that looks newer than its sources)."""
    src = PKG / "csrc" / "sg_api.cu"
    hdr = PKG.parent / "include" / "splinegpu.h"
    out = PKG / "libsplinegpu.so"
    stamp = PKG / "libsplinegpu.so.sha256"
    want = _source_hash(src, hdr)
    if not force and out.exists() and stamp.exists() and stamp.read_text().strip() == want:
        return out
    cmd = [str(NVCC), "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC", *ARCH, "-lineinfo",
           "-cudart", "static", "-o", str(out), str(src), f"-L{CUDA / 'lib64'}", "-lnvrtc",
           "-Xlinker", f"-rpath,{CUDA / 'lib64'}"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    stamp.write_text(want + "\n")
    return out


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
