"""Build a Part-I space with the per-reference-polynomial piece fits spread over processes
(the fits of different orbit representatives are independent).

    python tools/make_space_parallel.py bcc_voronoi3 [workers]
"""
import multiprocessing as mp
import pickle
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2102_08518_b200.model import SPACES_DIR, serialize_space, validate_space  # noqa: E402
from paper_2102_08518_b200.partone.make_spaces import BCC_COSETS, BCC_GEN, FCC_COSETS, FCC_GEN  # noqa: E402
from paper_2102_08518_b200.partone.producer import Producer  # noqa: E402
from paper_2102_08518_b200.partone.voronoi import BCC_VORONOI_GENS, FCC_VORONOI_GENS, voronoi_spline  # noqa: E402

SPECS = {
    "bcc_voronoi3": (lambda: voronoi_spline(BCC_VORONOI_GENS, 3), BCC_COSETS, BCC_GEN, (8, 8, 8)),
    "fcc_voronoi3": (lambda: voronoi_spline(FCC_VORONOI_GENS, 3), FCC_COSETS, FCC_GEN, (6, 6, 6)),
    "bcc_voronoi4": (lambda: voronoi_spline(BCC_VORONOI_GENS, 4), BCC_COSETS, BCC_GEN, (8, 8, 8)),
    "fcc_voronoi4": (lambda: voronoi_spline(FCC_VORONOI_GENS, 4), FCC_COSETS, FCC_GEN, (8, 8, 8)),
}
_P = None


def _fit_one(ri):
    p = _P
    p.reps = [p.reps_all[ri]]
    p.rng.seed(1000 + ri)
    polys = p.fit()
    return ri, polys[0], p.ref_stencils[0]


def main():
    global _P
    name = sys.argv[1]
    workers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    mk, cosets, gen, gext = SPECS[name]
    t0 = time.time()
    p = Producer(mk(), cosets, gen, name, "round_nearest", verbose=True)
    p.planes()
    p.regions()
    p.symmetries()
    p.orbits()
    p.reps_all = list(p.reps)
    _P = p
    # checkpoint of the fits, keyed by the representatives' sign vectors: a checkpoint from a
    # run whose orbit representatives differ must not be reused (it would attach every fit to
    # the wrong reference region)
    reps_key = [p.region_list[i].q for i in p.reps_all]
    ck = Path(f"/tmp/{name}_fits.pkl")
    res = None
    if ck.exists():
        saved = pickle.loads(ck.read_bytes())
        if isinstance(saved, dict) and saved.get("reps") == reps_key:
            res = saved["fits"]
    if res is None:
        with mp.get_context("fork").Pool(workers) as pool:
            res = sorted(pool.map(_fit_one, range(len(p.reps_all)), chunksize=1))
        ck.write_bytes(pickle.dumps({"reps": reps_key, "fits": res}))
    p.reps = p.reps_all
    p.ref_polys = [r[1] for r in res]
    p.ref_stencils = [r[2] for r in res]
    p.boundary_q()
    sp = p.assemble()
    errors = [d for d in validate_space(sp) if d.severity == "error"]
    if errors:
        raise SystemExit(f"{name}: {errors}")
    path = SPACES_DIR / f"{name}.json"
    path.write_text(serialize_space(sp, {"x_golden": {"extents": list(gext)}}))
    print(f"{path} in {time.time() - t0:.0f} s: {len(sp.subregions)} sub-regions, "
          f"K = {len(sp.ref_polys)}, n = {sp.stencil_size}", flush=True)


if __name__ == "__main__":
    main()
