"""Subsets of more than 128 frames (up to SR_MAX_FRAMES = 160): the paper's temporal schedule
build_temporal_levels(129, 17) ends with a 129-frame level.  The engine runs such subsets as 64-frame
blocks (pass 1 per block pair, one K x K finalize, pass 2 per block pair with the coefficients restricted
to it).  Checked against the oracle (fields, NCC and NGF, fp64 1e-10 / fp32 1e-4) and against the
reference package itself through the drop-in API (affine, fp64, 1e-10), including
seqreg.temporal.dissim_all_frames over 129 frames through install()."""

import numpy as np
import pytest
import torch

import paper_2001_06613_b200 as srb
from oracle import seqreg_oracle as orc
from tests.conftest import ref_types
from tests.test_parity_gpu import _frames_dev, _random_problem, _relmax

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("feature,dtype,K", [("ncc", torch.float64, 129), ("ngf", torch.float64, 129),
                                             ("ncc", torch.float32, 150), ("ngf", torch.float32, 129)])
def test_field_objective_large_k_matches_oracle(feature, dtype, K):
    rng = np.random.default_rng(K)
    dims = (20, 18)
    frames, spacing, origin, y, w = _random_problem(rng, dims, K, amp=0.3)
    h = float(np.prod(spacing))
    fd = _frames_dev(frames, dims, spacing, origin, dtype)
    obj = srb.FieldObjective(fd, list(range(K)), w, h, feature=feature, ngf_eps=0.5)
    yt = torch.as_tensor(y).to(device=fd.data.device, dtype=dtype).contiguous()
    stats, g = obj.evaluate(yt)
    D = float(stats[0].item())
    if dtype == torch.float32:
        frames = frames.astype(np.float32).astype(np.float64)
        y = y.astype(np.float32).astype(np.float64)
    st, Dref, gref = orc.evaluate_field(list(frames), dims, spacing, origin, y, w, h, feature, 0.5)
    tol = 1e-10 if dtype == torch.float64 else 1e-4
    assert D == pytest.approx(Dref, rel=tol)
    assert np.abs(obj.host_stats()["corr"] - st.corr).max() <= tol
    assert _relmax(g.double().cpu().numpy(), gref) < tol


def test_reference_api_129_frames_affine():
    from seqreg import similarity as ref_sim
    from seqreg import temporal as ref_tmp

    Grid, Image, ImageSequence, AffineStack = ref_types()
    rng = np.random.default_rng(7)
    dims, K = (16, 14), 129
    frames, spacing, origin, _, _ = _random_problem(rng, dims, K, amp=0.3)
    grid = Grid(dims, spacing, origin)
    times = np.linspace(0.0, 1.0, K)
    seq = ImageSequence([Image(grid, f) for f in frames], list(times))
    rows = np.tile(np.concatenate([np.eye(2).ravel(), np.zeros(2)]), (K, 1)) + 0.01 * rng.standard_normal((K, 6))
    subset = tuple(range(1, K + 1))
    stack = AffineStack.from_params(rows, subset, K, 2)
    w = ref_sim.quad_weights(times, *ref_sim.default_time_interval(times))
    st = srb.correlation_state(seq, stack, subset, w, grid.cell_volume)
    ref = ref_sim.correlation_state(seq, stack, subset, w, grid.cell_volume)
    assert np.abs(st.corr - ref.corr).max() <= 1e-12
    D, Dref = srb.dissimilarity(st), ref_sim.dissimilarity(ref)
    assert D == pytest.approx(Dref, rel=1e-10)
    g = srb.dissimilarity_gradient(st, seq, stack, subset)
    gref = ref_sim.dissimilarity_gradient(ref, seq, stack, subset)
    assert _relmax(g, gref) < 1e-10
    # the reference driver's all-frames score (temporal.py:297-301) through install()
    interval = ref_sim.default_time_interval(times)
    d_ref = ref_tmp.dissim_all_frames(seq, stack, interval, 1)
    srb.install()
    try:
        d_gpu = ref_tmp.dissim_all_frames(seq, stack, interval, 1)
    finally:
        srb.uninstall()
    assert d_gpu == pytest.approx(d_ref, rel=1e-10)


def test_more_than_max_frames_is_unsupported():
    rng = np.random.default_rng(1)
    from paper_2001_06613_b200._lib import SR_MAX_FRAMES

    dims, K = (8, 8), SR_MAX_FRAMES + 1
    frames, spacing, origin, y, w = _random_problem(rng, dims, K, amp=0.3)
    fd = _frames_dev(frames, dims, spacing, origin, torch.float64)
    obj = srb.FieldObjective(fd, list(range(K)), w, float(np.prod(spacing)))
    with pytest.raises(NotImplementedError):
        obj.evaluate(torch.as_tensor(y).to(device=fd.data.device).contiguous())
