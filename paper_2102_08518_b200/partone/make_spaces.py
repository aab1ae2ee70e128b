"""Write the package's shipped spaces (paper_2102_08518_b200/spaces/*.json).

    python -m paper_2102_08518_b200.partone.make_spaces [name ...]

Each file is the canonical serialization plus an `x_golden` key (ignored by
readers) giving the small extents tests/golden/make_golden.py uses.
"""

from __future__ import annotations

import sys

from ..model import SPACES_DIR, serialize_space, validate_space

BUILDERS = {}


def register(name, golden_extents):
    def deco(fn):
        BUILDERS[name] = (fn, golden_extents)
        return fn
    return deco


@register("tricubic", (8, 8, 8))
def _tricubic():
    from .tensor import tricubic
    return tricubic()


def write(name):
    fn, ext = BUILDERS[name]
    space = fn()
    errors = [d for d in validate_space(space) if d.severity == "error"]
    if errors:
        raise SystemExit(f"{name}: {errors}")
    SPACES_DIR.mkdir(exist_ok=True)
    path = SPACES_DIR / f"{name}.json"
    path.write_text(serialize_space(space, {"x_golden": {"extents": list(ext)}}))
    return path


def main(argv):
    names = argv or list(BUILDERS)
    for n in names:
        print(write(n))
    return 0


# -- box / Voronoi spline spaces built by the Part-I producer ---------------------------

from fractions import Fraction as _F  # noqa: E402

_H = _F(1, 2)
BCC_COSETS = [(0, 0, 0), (_H, _H, _H)]
BCC_GEN = [[1, 0, _H], [0, 1, _H], [0, 0, _H]]
BCC_DIRS = [(_H, _H, _H), (_H, -_H, -_H), (-_H, _H, -_H), (-_H, -_H, _H)]
FCC_COSETS = [(0, 0, 0), (_H, _H, 0), (_H, 0, _H), (0, _H, _H)]
FCC_GEN = [[_H, _H, 0], [_H, 0, _H], [0, _H, _H]]
FCC_DIRS = [(_H, _H, 0), (_H, -_H, 0), (_H, 0, _H), (_H, 0, -_H), (0, _H, _H), (0, _H, -_H)]


def _produce(phi, cosets, gen, name, rounding="round_nearest"):
    from .producer import Producer
    return Producer(phi, cosets, gen, name, rounding).run()


@register("bcc_box5", (8, 8, 8))
def _bcc_box5():
    """C2: BCC quintic box spline -- the 4 BCC nearest-neighbour directions, each twice."""
    from .boxspline import centered_box
    return _produce(centered_box(BCC_DIRS, [2, 2, 2, 2]), BCC_COSETS, BCC_GEN, "bcc_box5")


@register("bcc_box_linear", (8, 8, 8))
def _bcc_box_linear():
    """The BCC linear (rhombic-dodecahedron) box spline: the 4 directions once."""
    from .boxspline import centered_box
    return _produce(centered_box(BCC_DIRS), BCC_COSETS, BCC_GEN, "bcc_box_linear")


@register("fcc_box6", (6, 6, 6))
def _fcc_box6():
    """C4: FCC 6-direction (cubic truncated-octahedron) box spline."""
    from .boxspline import centered_box
    return _produce(centered_box(FCC_DIRS), FCC_COSETS, FCC_GEN, "fcc_box6")


@register("bcc_voronoi2", (8, 8, 8))
def _bcc_voronoi2():
    """C3/C5: BCC Voronoi spline of order 2 (truncated-octahedron cell convolved with
    itself; piecewise cubic), via the zonotopal tiling of the cell (voronoi.py)."""
    from .voronoi import BCC_VORONOI_GENS, voronoi_spline
    return _produce(voronoi_spline(BCC_VORONOI_GENS, 2), BCC_COSETS, BCC_GEN, "bcc_voronoi2")


@register("fcc_voronoi2", (6, 6, 6))
def _fcc_voronoi2():
    """FCC Voronoi spline of order 2 (rhombic-dodecahedron cell; piecewise cubic)."""
    from .voronoi import FCC_VORONOI_GENS, voronoi_spline
    return _produce(voronoi_spline(FCC_VORONOI_GENS, 2), FCC_COSETS, FCC_GEN, "fcc_voronoi2")


if __name__ == "__main__":
    raise SystemExit(main(sys.argv[1:]))
