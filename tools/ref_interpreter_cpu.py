"""CPU baseline path (2) of SURVEY 8d: the reference's generated-code evaluator
`interpret_batch(generate(space, GenConfig(ScheduleParams(1, n, "branchy"))), ...)` (the
paper's CPU default), timed on ONE core of the build container beside the
oracle port (oracle/refeval.py) on the same sample, so the GPU box's oracle-port numbers
(bench.py cpu_baseline / --impl reference) can be related to it.  Needs the reference
sources (/root/reference), so it runs here, not on the GPU box.

    python tools/ref_interpreter_cpu.py > profiles/r02_reference_interpreter_cpu.json
"""
import json
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import numpy as np  # noqa: E402

import bench  # noqa: E402
from oracle import refeval  # noqa: E402
from paper_2102_08518_b200.model import SPACES_DIR  # noqa: E402


def main():
    from splinegen.codegen import GenConfig, generate
    from splinegen.ir import DataVolume, interpret_batch
    from splinegen.model import InvariantError, parse_space
    from splinegen.schedule import ScheduleParams
    out = {"host": bench.cpu_model(), "cores_used": 1, "rows": []}
    seen = set()
    for cfg, c in bench.CONFIGS.items():
        name = c["space"]
        if name in seen:
            continue
        seen.add(name)
        text = (SPACES_DIR / f"{name}.json").read_text()
        osp = refeval.load_space_file(SPACES_DIR / f"{name}.json")
        rng = np.random.default_rng(0)
        ext = c["extents"]
        arrays = [rng.random(ext) for _ in range(osp.ncosets)]
        n = 2048
        xs = bench.make_queries(cfg, 0, n, "cpu").double().numpy()
        t0 = time.perf_counter()
        refeval.reference_eval_batch(osp, xs, arrays)
        t_or = time.perf_counter() - t0
        row = {"space": name, "config": cfg, "sample": n,
               "oracle_port_qps": n / t_or}
        try:
            sp = parse_space(text)
        except InvariantError as e:
            row["interpret_batch_qps"] = None
            row["note"] = ("the reference's generator refuses this space (" +
                           "; ".join(d.message for d in e.diagnostics if d.severity == "error")[:160] +
                           "): path (2) does not exist for it")
            out["rows"].append(row)
            print(json.dumps(row), file=sys.stderr)
            continue
        prog = generate(sp, GenConfig(ScheduleParams(1, sp.stencil_size, "branchy")))
        data = DataVolume(arrays)
        m = 512
        t0 = time.perf_counter()
        interpret_batch(prog, xs[:m], data)
        t_in = time.perf_counter() - t0
        row["interpret_batch_qps"] = m / t_in
        row["interpret_over_oracle"] = row["interpret_batch_qps"] / row["oracle_port_qps"]
        out["rows"].append(row)
        print(json.dumps(row), file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
