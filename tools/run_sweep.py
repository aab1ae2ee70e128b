"""Paper-style (m, d) x branch-mode sweep on the GPU: writes the
reference harness's CSV and lower-diagonal matrices for a few spaces into profiles/.

    python tools/run_sweep.py [space ...]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2102_08518_b200 import load_fixture, make_volume  # noqa: E402
from paper_2102_08518_b200.sweep import emit_csv, emit_matrix, run_sweep  # noqa: E402

EXTENTS = {"bcc_voronoi2": (101, 101, 101), "fcc_box6": (81, 81, 81), "zp_k2": (256, 256),
           "bcc_box5": (101, 101, 101),
           "trilinear_voronoi": (64, 64, 64), "bcc_box_linear": (101, 101, 101)}


def main():
    names = sys.argv[1:] or ["bcc_voronoi2", "fcc_box6", "bcc_box_linear"]
    for name in names:
        space = load_fixture(name)
        data = make_volume(space, EXTENTS[name], seed=0, float_width="f32")
        recs = run_sweep(space, data, trials=1 << 22, batch_size=1 << 20)
        out = ROOT / "profiles" / f"r01_sweep_{name}"
        out.with_suffix(".csv").write_text(emit_csv(recs))
        txt = [f"# {name}: mean reconstructions/s per (m, d) cell, rows d = 1.., columns m = 1..",
               "# (reference bench.py:82-215 lower-diagonal format; 2^22 uniform queries, f32, B200)"]
        for mode in ("predicated", "branchy"):
            txt.append(f"## {mode}")
            txt.append(emit_matrix(recs, mode))
        out.with_suffix(".txt").write_text("\n".join(txt) + "\n")
        best = max(recs, key=lambda r: r.mean_recon_per_sec)
        print(f"{name}: {len(recs)} cells, best m={best.m} d={best.d} {best.branch_mode} "
              f"{best.mean_recon_per_sec / 1e9:.2f} Grecon/s")


if __name__ == "__main__":
    main()
