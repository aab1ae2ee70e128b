import sys, torch, numpy as np
sys.path.insert(0, ".")
import bench
from paper_2102_08518_b200 import Evaluator, load_fixture, runtime
from paper_2102_08518_b200 import queries
space = load_fixture("bcc_voronoi2")
for E in [(101,101,101), (203,203,203)]:
    rng = np.random.default_rng(0)
    arrays = [rng.random(E).astype(np.float32) for _ in range(2)]
    for kind in ["uniform", "rays"]:
        n = 1 << 24
        xs = queries.uniform(0, n, E, 1, "cuda") if kind == "uniform" else queries.rays(0, n, E, 512, 512, 64, 2, "cuda")
        for mode in ["direct", "sorted"]:
            kw = dict(mode=mode, block=512 if mode=="sorted" else 128)
            _, prog = bench.build_program("c3", **kw) if E == (203,203,203) else (None, None)
            if prog is None:
                from paper_2102_08518_b200 import generate
                prog = generate(space, bench.gen_config_for(space, False, coeffs="imm", **kw), E)
            ev = Evaluator(space, arrays, prog=prog)
            out = torch.empty(n, device="cuda")
            for _ in range(3): runtime.eval_device(ev.module, ev.volume, xs, out)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(10): runtime.eval_device(ev.module, ev.volume, xs, out)
            b.record(); torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 10
            print(E[0], kind, mode, f"{ms:.3f} ms  {n/ms/1e6:.2f} Grecon/s", flush=True)
