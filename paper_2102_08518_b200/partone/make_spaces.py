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


if __name__ == "__main__":
    raise SystemExit(main(sys.argv[1:]))
