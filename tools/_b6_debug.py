import sys; sys.path.insert(0,'/root/repo')
import torch, bench
from paper_2102_08518_b200 import Evaluator, GenConfig, ScheduleParams, generate, load_fixture
from paper_2102_08518_b200 import runtime
import numpy as np
space, arrays, xs = bench.make_inputs("c2", 0, torch.device("cuda",0))
xs = xs[:1<<16].contiguous()
ref = None
for b in (8, 4, 12, 16, 20):
    for stage in ("tma", "ldg"):
        try:
            _, prog = bench.build_program("c2", mode="binned", stage=stage, block=256, unroll_cosets=False, bin=b)
            ev = Evaluator(space, arrays, prog=prog)
            out = ev(xs)
            torch.cuda.synchronize()
            if ref is None: ref = out.clone()
            print("bin", b, stage, "brick", prog.brick, "ok", float((out-ref).abs().max()), flush=True)
        except Exception as e:
            print("bin", b, stage, "brick", prog.brick, "FAIL", str(e)[:100], flush=True)
            sys.exit(0)
