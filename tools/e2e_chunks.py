"""End-to-end (host buffers, sg_eval_host) rate of a bench config for several chunk sizes.

    python tools/e2e_chunks.py c2
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2102_08518_b200 import Evaluator, runtime  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
dev = torch.device("cuda", 0)
space, arrays, xs = bench.make_inputs(cfg, 0, dev)
_, prog = bench.build_program(cfg)
ev = Evaluator(space, arrays, prog=prog)
n = xs.shape[0]
xh = xs.cpu().pin_memory()
oh = torch.empty(n, dtype=torch.float32).pin_memory()
gh = torch.empty((n, space.dim), dtype=torch.float32).pin_memory() if prog.has_grad else None
lib = runtime.lib()
for lg in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else "20,21,22,23,24".split(","))]:
    chunk = 1 << lg

    def step():
        runtime._check(lib.sg_eval_host(ev.module.handle, ev.volume.handle,
                                        runtime.ctypes.c_void_p(xh.data_ptr()), n,
                                        runtime.ctypes.c_void_p(oh.data_ptr()),
                                        runtime.ctypes.c_void_p(gh.data_ptr() if gh is not None else 0),
                                        chunk))
    step()
    t0 = time.perf_counter()
    for _ in range(10):
        step()
    dt = (time.perf_counter() - t0) / 10
    print(f"chunk 2^{lg}: {dt * 1e3:.2f} ms/step  {n / dt / 1e9:.3f} Grecon/s  "
          f"H2D {n * space.dim * 4 / dt / 1e9:.1f} GB/s", flush=True)
