"""The C ABI from plain C (examples/capi_demo.c, gcc): compile a generated kernel with
sg_compile, load it, upload a volume, evaluate a batch through sg_eval_host, and compare
with the oracle -- no Python or torch on the evaluation path."""

import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import refeval
from tests.gpu_util import ATOL_F32, RTOL_F32, close, load_golden

ROOT = Path(__file__).resolve().parents[1]


def _build(tmp):
    exe = tmp / "capi_demo"
    lib = ROOT / "paper_2102_08518_b200"
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-o", str(exe), str(ROOT / "examples" / "capi_demo.c"),
                    f"-L{lib}", "-lsplinegpu", f"-Wl,-rpath,{lib}"], check=True)
    return exe


def test_capi_demo_builds_with_gcc(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
@pytest.mark.parametrize("name,mode", [("bcc_box5", "binned"), ("bcc_voronoi2", "direct"),
                                       ("tricubic", "binned")])
def test_capi_demo_matches_oracle(tmp_path, name, mode):
    from paper_2102_08518_b200 import GenConfig, ScheduleParams, generate
    space, ospace, z, arrays = load_golden(name)
    prog = generate(space, GenConfig(ScheduleParams(1, space.stencil_size), mode=mode,
                                     float_width="f32"),
                    arrays[0].shape)
    (tmp_path / "k.cu").write_text(prog.source)
    fields = [prog.dim, prog.ncosets, prog.block, prog.halo, 1 if prog.mode == "binned" else 0,
              prog.rounding, int(prog.stage_tma), prog.smem_bytes, prog.bin, prog.chunk]
    fields += [e for row in prog.padded_extents for e in row]
    fields += list(prog.extents[0]) + (list(prog.brick) or [0] * prog.dim)
    (tmp_path / "info.txt").write_text(" ".join(str(int(v)) for v in fields) + "\n")
    np.concatenate([a.astype(np.float32).ravel() for a in arrays]).tofile(tmp_path / "vol.bin")
    xs = z["uniform_xs"].astype(np.float32)
    xs.tofile(tmp_path / "q.bin")
    exe = _build(tmp_path)
    r = subprocess.run([str(exe), str(tmp_path / "k.cu"), str(tmp_path / "info.txt"),
                        str(tmp_path / "vol.bin"), str(tmp_path / "q.bin"), str(tmp_path / "out.bin")],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = np.fromfile(tmp_path / "out.bin", dtype=np.float32).astype(np.float64)
    want = refeval.reference_eval_batch(ospace, xs.astype(np.float64), [a.astype(np.float64) for a in arrays])
    assert close(got, want, RTOL_F32, ATOL_F32).all()
