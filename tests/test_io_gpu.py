"""GPU: STSQ1 files straight to HBM (paper_2001_06613_b200.io) against the reference reader's
values (tests/golden/stsq1_golden.npz) and writer's bytes (tests/golden/small_seq.stsq1); and the
report's dissim_all_frames (temporal.py:297-301) through install()."""

from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2001_06613_b200 as srb
from paper_2001_06613_b200 import io as sio

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
REF = np.load(GOLD / "stsq1_golden.npz")


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_read_sequence_matches_reference(dtype):
    fd, times = sio.read_sequence(GOLD / "small_seq.stsq1", dtype=dtype)
    assert fd.data.is_cuda and fd.data.dtype == dtype
    assert tuple(fd.grid.dims) == tuple(REF["dims"])
    assert tuple(fd.grid.spacing) == tuple(REF["spacing"]) and tuple(fd.grid.origin) == tuple(REF["origin"])
    assert times == list(REF["times"])
    got = fd.data.cpu().numpy()
    want = REF["values"] if dtype == torch.float64 else REF["values"].astype(np.float32)
    np.testing.assert_array_equal(got, want)


def test_write_sequence_is_byte_identical(tmp_path):
    fd, times = sio.read_sequence(GOLD / "small_seq.stsq1")
    out = tmp_path / "rt.stsq1"
    sio.write_sequence(fd, times, out)
    assert out.read_bytes() == (GOLD / "small_seq.stsq1").read_bytes()


def test_large_round_trip(tmp_path):
    grid = srb.GridSpec((256, 192), (1 / 256, 1 / 192), (0.0, 0.0))
    data = torch.randn((5, grid.cell_count), device="cuda", dtype=torch.float32)
    fd = srb.DeviceFrames(srb.get_engine(), data, grid)
    p = tmp_path / "big.stsq1"
    sio.write_sequence(fd, [0.0, 0.25, 0.5, 0.75, 1.0], p)
    back, t = sio.read_sequence(p, dtype=torch.float32)
    assert torch.equal(back.data, data) and t == [0.0, 0.25, 0.5, 0.75, 1.0]
