"""Writes a small sequence with the reference's writer (seqreg.grid.write_sequence, grid.py:256-268),
records what the reference reader returns for it and the exception class / message it raises for
each malformed variant of tests/stsq1_cases.py.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_stsq1_golden.py
"""

import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from seqreg.grid import Grid, Image, ImageSequence, read_sequence, write_sequence  # noqa: E402

from tests.stsq1_cases import variants  # noqa: E402


def main():
    rng = np.random.default_rng(7)
    grid = Grid((9, 7), (0.5, 0.25), (-1.25, 0.1))
    vals = rng.standard_normal((3, grid.cell_count)) * 3.0
    seq = ImageSequence([Image(grid, v) for v in vals], [0.0, 1.0 / 3.0, 0.37])
    out = ROOT / "tests" / "golden" / "small_seq.stsq1"
    write_sequence(seq, out)
    back = read_sequence(out)
    np.savez_compressed(ROOT / "tests" / "golden" / "stsq1_golden.npz",
                        values=np.stack([f.values for f in back.frames]), times=np.array(back.times),
                        dims=np.array(back.grid.dims), spacing=np.array(back.grid.spacing),
                        origin=np.array(back.grid.origin))
    errors = {}
    with tempfile.TemporaryDirectory() as td:
        for name, data in variants(out.read_bytes()).items():
            p = Path(td) / f"{name}.stsq1"
            p.write_bytes(data)
            try:
                read_sequence(p)
                errors[name] = None
            except Exception as exc:  # record the reference's behaviour verbatim
                errors[name] = [type(exc).__name__, str(exc)]
    (ROOT / "tests" / "golden" / "stsq1_errors.json").write_text(json.dumps(errors, indent=1))
    print(json.dumps(errors, indent=1))


if __name__ == "__main__":
    main()
