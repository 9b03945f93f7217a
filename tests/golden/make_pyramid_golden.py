"""Runs the reference pyramid (seqreg.pyramid.build_pyramid, pyramid.py:68-91) on small seeded
2-D / 3-D sequences with odd axes and writes tests/golden/pyramid_golden.npz.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_pyramid_golden.py
"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, "/root/reference/pkg/src")

from seqreg.grid import Grid, Image, ImageSequence  # noqa: E402
from seqreg.pyramid import build_pyramid  # noqa: E402

CASES = {"p2d": ((37, 29), (0.5, 0.25), (-3.0, 1.0), 3, 3), "p3d": ((13, 10, 9), (1.0, 0.5, 2.0), (0.0, 0.0, 0.0), 2, 2)}


def main():
    out = {}
    for name, (dims, spacing, origin, nframes, levels) in CASES.items():
        rng = np.random.default_rng(len(dims))
        grid = Grid(dims, spacing, origin)
        vals = rng.standard_normal((nframes, grid.cell_count)) * 10.0 ** rng.uniform(-2, 2, (nframes, 1))
        seq = ImageSequence([Image(grid, v) for v in vals], list(range(nframes)))
        pyr = build_pyramid(seq, levels)
        out[f"{name}_input"] = vals
        out[f"{name}_meta"] = np.array([len(dims), *dims, *([1] * (3 - len(dims))), levels, nframes])
        out[f"{name}_spacing"] = np.array(spacing)
        out[f"{name}_origin"] = np.array(origin)
        for lv, s in enumerate(pyr.levels):
            out[f"{name}_level{lv}"] = np.stack([f.values for f in s.frames])
            out[f"{name}_level{lv}_dims"] = np.array(s.grid.dims)
            out[f"{name}_level{lv}_spacing"] = np.array(s.grid.spacing)
        print(name, [s.grid.dims for s in pyr.levels])
    np.savez_compressed(ROOT / "tests" / "golden" / "pyramid_golden.npz", **out)


if __name__ == "__main__":
    main()
