"""GPU: sr_pyramid_step / build_pyramid against the reference's levels (fp64 bit-identical, fp32
within 1e-6 relative) and sr_prolong_field against the oracle."""

from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2001_06613_b200 as srb
from oracle import seqreg_oracle as orc

pytestmark = pytest.mark.gpu

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "pyramid_golden.npz")


def _frames(name, dtype):
    m = GOLD[f"{name}_meta"]
    nd = int(m[0])
    dims = tuple(int(v) for v in m[1:1 + nd])
    grid = srb.GridSpec(dims, tuple(GOLD[f"{name}_spacing"]), tuple(GOLD[f"{name}_origin"]))
    data = torch.as_tensor(GOLD[f"{name}_input"], dtype=dtype, device="cuda")
    return srb.DeviceFrames(srb.get_engine(), data, grid), int(m[4])


@pytest.mark.parametrize("name", ["p2d", "p3d"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_build_pyramid_matches_reference(name, dtype):
    fd, levels = _frames(name, dtype)
    pyr = srb.build_pyramid(fd, levels)
    assert len(pyr) == levels and pyr[-1] is fd
    for lv in range(levels - 1):
        got = pyr[lv].data.double().cpu().numpy()
        want = GOLD[f"{name}_level{lv}"]
        assert tuple(pyr[lv].grid.dims) == tuple(GOLD[f"{name}_level{lv}_dims"])
        np.testing.assert_array_equal(np.asarray(pyr[lv].grid.spacing), GOLD[f"{name}_level{lv}_spacing"])
        if dtype == torch.float64:
            np.testing.assert_array_equal(got, want)
        else:
            assert np.abs(got - want).max() <= 1e-6 * np.abs(want).max()


def test_build_pyramid_validation():
    fd, _ = _frames("p2d", torch.float64)
    with pytest.raises(ValueError, match="level_count must be >= 1"):
        srb.build_pyramid(fd, 0)
    with pytest.raises(ValueError, match="too large for dims"):
        srb.build_pyramid(fd, 5)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("cdims,fdims", [((6, 5), (12, 10)), ((7, 5), (13, 9)), ((4, 5, 3), (8, 9, 6))])
def test_prolong_field_vs_oracle(dtype, cdims, fdims):
    d = len(cdims)
    rng = np.random.default_rng(d * 100 + cdims[0])
    cs = tuple(rng.uniform(0.3, 1.0, d))
    fs = tuple(s / 2 for s in cs)
    o = tuple(rng.uniform(-1, 1, d))
    k = 3
    xc = orc.cell_centers(cdims, cs, o).T
    yc = xc[None] + 0.2 * rng.standard_normal((k, d, xc.shape[1])) * np.asarray(cs)[None, :, None]
    want = orc.prolong_field(yc, cdims, cs, o, fdims, fs, o)
    got = srb.prolong_field(torch.as_tensor(yc, dtype=dtype, device="cuda"), srb.GridSpec(cdims, cs, o),
                            srb.GridSpec(fdims, fs, o))
    tol = 1e-13 if dtype == torch.float64 else 2e-6
    assert np.abs(got.double().cpu().numpy() - want).max() <= tol * max(1.0, np.abs(want).max())
