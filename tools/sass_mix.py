"""Static SASS instruction mix of a bench config's evaluation kernel.

    python tools/sass_mix.py c3 [key=value ...]     (variant overrides, e.g. form=sym)
"""
import collections
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2102_08518_b200.runtime import compile_source  # noqa: E402


def mix(cubin: bytes):
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(cubin)
        f.flush()
        txt = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
    ops = collections.Counter()
    for ln in txt.splitlines():
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
        if m:
            ops[m.group(2).split(".")[0]] += 1
    return ops, txt


def main():
    cfg = sys.argv[1]
    over = {}
    for kv in sys.argv[2:]:
        k, v = kv.split("=")
        over[k] = int(v) if v.isdigit() else v
    _, prog = bench.build_program(cfg, **over)
    img, key = compile_source(prog.source)
    ops, txt = mix(img)
    tot = sum(ops.values())
    print(f"{cfg} {over} total {tot} SASS instructions")
    for op, c in ops.most_common(40):
        print(f"  {op:10s} {c:6d}")


if __name__ == "__main__":
    main()
