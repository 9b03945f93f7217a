"""CPU: the pyramid restatement (oracle) reproduces the reference's build_pyramid bit for bit
(tests/golden/pyramid_golden.npz), and the prolongation oracle's defining properties hold."""

from pathlib import Path

import numpy as np
import pytest

from oracle import seqreg_oracle as orc

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "pyramid_golden.npz")


def _meta(name):
    m = GOLD[f"{name}_meta"]
    nd = int(m[0])
    return nd, tuple(int(v) for v in m[1:1 + nd]), int(m[4]), int(m[5])


@pytest.mark.parametrize("name", ["p2d", "p3d"])
def test_oracle_pyramid_matches_reference(name):
    nd, dims, levels, nframes = _meta(name)
    cur = GOLD[f"{name}_input"]
    cdims = dims
    for lv in range(levels - 2, -1, -1):  # golden levels are coarse to fine; the finest is the input
        nxt = []
        for f in cur:
            v, cdims2 = orc.pyramid_step_flat(f, cdims)
            nxt.append(v)
        cur, cdims = np.stack(nxt), cdims2
        np.testing.assert_array_equal(cur, GOLD[f"{name}_level{lv}"])
        assert tuple(cdims) == tuple(GOLD[f"{name}_level{lv}_dims"])


def test_prolong_oracle_properties():
    cdims, cs, co = (6, 5), (0.4, 0.6), (-1.0, 0.5)
    fdims, fs = (12, 10), (0.2, 0.3)
    xc = orc.cell_centers(cdims, cs, co).T
    # a constant displacement is carried exactly
    y = xc[None] + np.array([0.03, -0.02])[None, :, None]
    yf = orc.prolong_field(y, cdims, cs, co, fdims, fs, co)
    xf = orc.cell_centers(fdims, fs, co).T
    np.testing.assert_allclose(yf - xf[None], np.broadcast_to(np.array([0.03, -0.02])[None, :, None], yf.shape),
                               atol=1e-14)
    # an affine displacement is carried exactly inside the hull of the coarse centres
    A = np.array([[0.01, 0.02], [-0.03, 0.015]])
    y = xc[None] + (A @ xc)[None]
    yf = orc.prolong_field(y, cdims, cs, co, fdims, fs, co)
    lo, hi = xc.min(axis=1), xc.max(axis=1)
    inside = np.all((xf >= lo[:, None]) & (xf <= hi[:, None]), axis=0)
    np.testing.assert_allclose((yf - xf[None])[0][:, inside], (A @ xf)[:, inside], atol=1e-14)
