"""GPU parity tests: the CUDA path (through the C-ABI) against the reference's golden
vectors and the oracle.  Tolerances (north_star): 1e-10 relative in fp64, 1e-4 in fp32.
Relative gradient errors are measured against the largest gradient entry."""

import zlib

import numpy as np
import pytest
import torch

import paper_2001_06613_b200 as srb
from oracle import seqreg_oracle as orc
from tests.conftest import golden_frames, ref_types

pytestmark = pytest.mark.gpu

AFFINE_CASES = [
    "aff2d_small_0", "aff2d_small_1", "aff2d_small_2", "aff2d_identity_dyadic", "aff2d_identity_nondyadic",
    "aff2d_subset_outside", "aff3d_small", "aff2d_degenerate", "c1_identity", "c1_perturbed", "c1_subset",
]
TOL = {torch.float64: 1e-10, torch.float32: 1e-4}


def _relmax(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def _seq_stack(case):
    Grid, Image, ImageSequence, AffineStack = ref_types()
    frames = golden_frames(case)
    grid = Grid(tuple(case["dims"]), tuple(case["spacing"]), tuple(case["origin"]))
    seq = ImageSequence([Image(grid, f) for f in frames], list(case["times"]))
    subset = tuple(int(k) for k in case["subset"])
    stack = AffineStack.from_params(case["rows"], subset, len(frames), grid.ndim)
    return seq, stack, subset


@pytest.fixture(autouse=True)
def _reset_options():
    srb.configure(dtype=torch.float64, feature="ncc")
    yield
    srb.configure(dtype=torch.float64, feature="ncc")


@pytest.mark.parametrize("name", AFFINE_CASES)
def test_affine_reference_api_fp64_matches_reference(golden, name):
    """The drop-in trio reproduces seqreg's correlation_state / dissimilarity / gradient."""
    case = golden[name]
    seq, stack, subset = _seq_stack(case)
    st = srb.correlation_state(seq, stack, subset, case["weights"], float(case["h"]))
    np.testing.assert_allclose(st.corr, case["corr"], rtol=0, atol=1e-12)
    assert np.array_equal(st.corr, st.corr.T)
    assert np.array_equal(st.degenerate, case["degenerate"])
    D = srb.dissimilarity(st)
    assert D == pytest.approx(float(case["D"]), rel=1e-10, abs=1e-13)
    g = srb.dissimilarity_gradient(st, seq, stack, subset)
    assert g.shape == case["grad"].shape
    assert _relmax(g, case["grad"]) < 1e-10
    nd = ~case["degenerate"]
    np.testing.assert_allclose(st.center_norms[nd], case["center_norms"][nd], rtol=1e-10)


@pytest.mark.parametrize("name", ["aff2d_small_0", "aff2d_identity_dyadic", "aff3d_small", "c1_perturbed"])
def test_affine_reference_api_fp32(golden, name):
    case = golden[name]
    seq, stack, subset = _seq_stack(case)
    srb.configure(dtype=torch.float32)
    st = srb.correlation_state(seq, stack, subset, case["weights"], float(case["h"]))
    D = srb.dissimilarity(st)
    g = srb.dissimilarity_gradient(st, seq, stack, subset)
    # oracle on the same fp32-quantised frames, evaluated in fp64
    frames = golden_frames(case).astype(np.float32).astype(np.float64)
    fr = [frames[k - 1] for k in subset]
    _, Dref, gref = orc.evaluate_affine(fr, tuple(case["dims"]), tuple(case["spacing"]), tuple(case["origin"]),
                                        case["rows"], case["weights"], float(case["h"]))
    assert D == pytest.approx(Dref, rel=1e-4)
    assert _relmax(g, gref) < 1e-4


def test_reference_api_errors(golden):
    case = golden["aff2d_small_0"]
    seq, stack, subset = _seq_stack(case)
    with pytest.raises(ValueError, match="nonempty"):
        srb.correlation_state(seq, stack, (), [], 1.0)
    with pytest.raises(ValueError, match="strictly increasing"):
        srb.correlation_state(seq, stack, (2, 1), [0.5, 0.5], 1.0)
    with pytest.raises(ValueError, match="one weight"):
        srb.correlation_state(seq, stack, subset, [1.0], 1.0)
    st = srb.correlation_state(seq, stack, subset, case["weights"], 1.0)
    with pytest.raises(ValueError, match="does not match"):
        srb.dissimilarity_gradient(st, seq, stack, (1, 2))


def _frames_dev(frames_np, dims, spacing, origin, dtype):
    eng = srb.get_engine()
    return srb.DeviceFrames.from_array(eng, np.asarray(frames_np), srb.GridSpec(tuple(dims), tuple(spacing),
                                                                                  tuple(origin)), dtype)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_displacement_affine_contraction_matches_reference(golden, dtype):
    """y_k(x) = A_k x + b_k as a displacement field: D equals the reference's, and the
    per-cell gradient contracted with [x, 1] equals its affine gradient."""
    for name in ["aff2d_small_1", "aff2d_subset_outside", "aff3d_small", "c1_perturbed"]:
        case = golden[name]
        dims, sp, org = tuple(case["dims"]), tuple(case["spacing"]), tuple(case["origin"])
        frames = golden_frames(case)
        subset0 = [int(k) - 1 for k in case["subset"]]
        x = orc.cell_centers(dims, sp, org)
        y = np.stack([orc.affine_points(r, x).T for r in case["rows"]])
        fd = _frames_dev(frames, dims, sp, org, dtype)
        obj = srb.FieldObjective(fd, subset0, case["weights"], float(case["h"]))
        yt = torch.as_tensor(y).to(device=fd.data.device, dtype=dtype).contiguous()
        stats, g = obj.evaluate(yt)
        D = float(stats[0].item())
        gy = g.double().cpu().numpy()
        rows = np.array([np.concatenate([(gk @ x).ravel(), gk.sum(axis=1)]) for gk in gy])
        if dtype == torch.float64:
            assert D == pytest.approx(float(case["D"]), rel=1e-10, abs=1e-13), name
            assert _relmax(rows, case["grad"]) < 1e-10, name
        else:
            q = frames.astype(np.float32).astype(np.float64)
            yq = y.astype(np.float32).astype(np.float64)
            _, Dref, gref = orc.evaluate_field([q[k] for k in subset0], dims, sp, org, yq, case["weights"],
                                               float(case["h"]))
            assert D == pytest.approx(Dref, rel=1e-4), name
            assert _relmax(gy, gref) < 1e-4, name


def _random_problem(rng, dims, K, amp=0.4, nframes=None):
    from scipy.ndimage import gaussian_filter
    d = len(dims)
    spacing = tuple([0.5, 0.25, 0.75][:d])
    origin = tuple(-n * s / 2 for n, s in zip(dims, spacing))
    nframes = nframes or K
    frames = np.stack([gaussian_filter(rng.standard_normal(dims), 1.5, mode="reflect").ravel(order="F") + 3.0
                       for _ in range(nframes)])
    x = orc.cell_centers(dims, spacing, origin).T
    y = x[None] + amp * rng.standard_normal((K,) + x.shape) * np.asarray(spacing)[None, :, None]
    # keep samples off grid nodes: there the interpolant's derivative jumps, and an fp32 rounding of y
    # can flip the cell (the kink hazard, pinned separately by test_identity_kink_gradient_fp32_dyadic)
    s_, o_ = np.asarray(spacing)[None, :, None], np.asarray(origin)[None, :, None]
    t_ = (y - o_) / s_ - 0.5
    fr = t_ - np.floor(t_)
    y = np.where((fr < 2e-3) | (fr > 1 - 2e-3), y + 5e-3 * s_, y)
    w = rng.uniform(0.5, 1.0, K)
    return frames, spacing, origin, y, w


@pytest.mark.parametrize("feature", ["ncc", "ngf"])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("dims,K", [((24, 20), 3), ((33, 17), 12), ((20, 18), 27), ((16, 12), 40),
                                    ((12, 10), 100), ((10, 9, 8), 5), ((9, 8, 7), 20)])
def test_field_parity_vs_oracle(feature, dtype, dims, K):
    """Displacement-field D and dD/dy vs the oracle, every KP bucket, 2-D and 3-D."""
    rng = np.random.default_rng(zlib.crc32(repr((feature, str(dtype), dims, K)).encode()))
    frames, spacing, origin, y, w = _random_problem(rng, dims, K, nframes=K + 2)
    subset0 = sorted(rng.choice(K + 2, size=K, replace=False).tolist())
    h = float(np.prod(spacing))
    fd = _frames_dev(frames, dims, spacing, origin, dtype)
    obj = srb.FieldObjective(fd, subset0, w, h, feature=feature, ngf_eps=0.2)
    yt = torch.as_tensor(y).to(device=fd.data.device, dtype=dtype).contiguous()
    stats, g = obj.evaluate(yt)
    D = float(stats[0].item())
    q = frames if dtype == torch.float64 else frames.astype(np.float32).astype(np.float64)
    yq = y if dtype == torch.float64 else y.astype(np.float32).astype(np.float64)
    st, Dref, gref = orc.evaluate_field([q[k] for k in subset0], dims, spacing, origin, yq, w, h, feature, 0.2)
    tol = TOL[dtype]
    hs = obj.host_stats()
    np.testing.assert_allclose(hs["corr"], st.corr, rtol=0, atol=tol)
    assert D == pytest.approx(Dref, rel=tol)
    assert _relmax(g.double().cpu().numpy(), gref) < tol


@pytest.mark.parametrize("feature", ["ncc", "ngf"])
def test_ngf_ncc_affine_fp64_vs_oracle(golden, feature):
    case = golden["aff2d_subset_outside"]
    seq, stack, subset = _seq_stack(case)
    srb.configure(feature=feature, ngf_eps=0.3)
    st = srb.correlation_state(seq, stack, subset, case["weights"], float(case["h"]))
    g = srb.dissimilarity_gradient(st, seq, stack, subset)
    frames = golden_frames(case)
    ost, Dref, gref = orc.evaluate_affine([frames[k - 1] for k in subset], tuple(case["dims"]),
                                          tuple(case["spacing"]), tuple(case["origin"]), case["rows"],
                                          case["weights"], float(case["h"]), feature, 0.3)
    np.testing.assert_allclose(st.corr, ost.corr, rtol=0, atol=1e-12)
    assert srb.dissimilarity(st) == pytest.approx(Dref, rel=1e-10)
    assert _relmax(g, gref) < 1e-10


def test_identity_kink_gradient_fp32_dyadic(golden):
    """At the identity every sample is a node: fp32 t must pick the right-sided cell like the
    reference; compare against the fp64 reference gradient with fp32 tolerance."""
    case = golden["aff2d_identity_dyadic"]
    dims, sp, org = tuple(case["dims"]), tuple(case["spacing"]), tuple(case["origin"])
    frames = golden_frames(case)
    x = orc.cell_centers(dims, sp, org)
    y = np.stack([x.T for _ in case["rows"]])
    fd = _frames_dev(frames, dims, sp, org, torch.float32)
    obj = srb.FieldObjective(fd, [int(k) - 1 for k in case["subset"]], case["weights"], float(case["h"]))
    _, g = obj.evaluate(torch.as_tensor(y, dtype=torch.float32, device=fd.data.device).contiguous())
    gy = g.double().cpu().numpy()
    rows = np.array([np.concatenate([(gk @ x).ravel(), gk.sum(axis=1)]) for gk in gy])
    assert _relmax(rows, case["grad"]) < 1e-4


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
@pytest.mark.parametrize("dims", [(17, 13), (9, 8, 7)])
def test_curvature_vs_oracle(dtype, dims):
    rng = np.random.default_rng(11)
    frames, spacing, origin, y, w = _random_problem(rng, dims, 3, amp=0.3)
    h = float(np.prod(spacing))
    fd = _frames_dev(frames, dims, spacing, origin, dtype)
    obj = srb.FieldObjective(fd, [0, 1, 2], w, h, alpha=2.5)
    obj0 = srb.FieldObjective(fd, [0, 1, 2], w, h)
    yt = torch.as_tensor(y).to(device=fd.data.device, dtype=dtype).contiguous()
    _, g = obj.evaluate(yt)
    _, g0 = obj0.evaluate(yt)
    S = float(obj.s_reg.item())
    Sref, gS = orc.curvature(y if dtype == torch.float64 else y.astype(np.float32).astype(np.float64),
                             dims, spacing, origin, 2.5, h)
    assert S == pytest.approx(Sref, rel=TOL[dtype] * 10)
    assert _relmax((g - g0).double().cpu().numpy(), gS) < TOL[dtype] * 10


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_temporal_vs_reference(golden, dtype):
    c = golden["temporal"]
    n = c["ref"].shape[0]
    active0 = [int(k) - 1 for k in c["active"]]
    eta = np.zeros_like(c["ref"])
    eta[active0] = c["eta"]
    mask = np.zeros(n, bool)
    mask[active0] = True
    dev = torch.device("cuda")
    z = srb.ls_predict_fields(torch.as_tensor(eta, dtype=dtype, device=dev), mask,
                              torch.as_tensor(c["ref"], dtype=dtype, device=dev), float(c["beta"]))
    tol = 1e-13 if dtype == torch.float64 else 1e-5
    np.testing.assert_allclose(z.double().cpu().numpy(), c["ls"], rtol=0, atol=tol * np.abs(c["ls"]).max())
    lin = srb.interp_linear_fields(torch.as_tensor(eta, dtype=dtype, device=dev), active0, c["times"])
    np.testing.assert_allclose(lin.double().cpu().numpy(), c["interp"], rtol=0, atol=tol)


def test_temporal_fields_large_vs_oracle():
    rng = np.random.default_rng(8)
    n, m = 17, 5000
    ref = rng.standard_normal((n, m))
    mask = np.zeros(n, bool)
    mask[::4] = True
    mask[-1] = True
    eta = rng.standard_normal((n, m))
    dev = torch.device("cuda")
    z = srb.ls_predict_fields(torch.as_tensor(eta, device=dev), mask, torch.as_tensor(ref, device=dev), 2.0)
    zr = orc.ls_predict_arrays(eta, mask, ref, 2.0)
    assert _relmax(z.cpu().numpy(), zr) < 1e-12
    with pytest.raises(ValueError):
        srb.ls_predict_fields(torch.as_tensor(eta, device=dev), mask, torch.as_tensor(ref, device=dev), 0.0)


@pytest.mark.parametrize("feature", ["ncc", "ngf"])
def test_slab_sharding_sums_to_whole(feature):
    """Pixel slabs (the multi-GPU partition) reduce to the whole-grid evaluation: raw sums add
    up, and the per-slab gradients tile the whole gradient (NGF needs the 1-row halo)."""
    rng = np.random.default_rng(21)
    dims, K = (40, 24), 6
    frames, spacing, origin, y, w = _random_problem(rng, dims, K)
    h = float(np.prod(spacing))
    fd = _frames_dev(frames, dims, spacing, origin, torch.float64)
    whole = srb.FieldObjective(fd, list(range(K)), w, h, feature=feature, ngf_eps=0.2)
    yt = torch.as_tensor(y, device=fd.data.device).contiguous()
    stats, g = whole.evaluate(yt)
    N = int(np.prod(dims))
    row = dims[0]
    cuts = [0, 7 * row, 16 * row, N]
    raws = []
    plans = []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        plan = srb.EvalPlan(fd, list(range(K)), feature=feature, ngf_eps=0.2, pix_range=(lo, hi))
        prob = plan.problem(y=yt)
        raws.append(plan.corr_partial(prob).clone())
        plans.append((plan, prob, lo, hi))
    total = sum(raws)
    ext = torch.stack([r[K * K + K:K * K + 3 * K] for r in raws]).amax(0)
    total[K * K + K:K * K + 3 * K] = ext
    assert int(total[-1].item()) == N
    gs = torch.zeros_like(yt)
    for plan, prob, lo, hi in plans:
        plan.raw.copy_(total)
        plan.finalize(prob, w, h, n_total=N)
        assert float(plan.stats[0].item()) == pytest.approx(float(stats[0].item()), rel=1e-12)
        out = torch.empty((K, 2, hi - lo), dtype=yt.dtype, device=yt.device)
        plan.grad(prob, out, g_off=lo)
        gs[:, :, lo:hi] = out
    assert _relmax(gs.cpu().numpy(), g.cpu().numpy()) < 1e-12


@pytest.mark.parametrize("reuse", [False, True])
@pytest.mark.parametrize("feature", ["ncc", "ngf"])
@pytest.mark.parametrize("dims", [(40, 24), (37, 26)])
def test_slab_sharding_fp32_tensor_core_path(feature, dims, reuse):
    """The fp32 K <= 32 split path (pipelined sampler, TMA-fed Gram, TMA-fed pass 2 / NGF z) on pixel
    slabs — including slab starts that are not 16-byte aligned — reduces to the whole-grid evaluation
    (fp32: summation order differs, 1e-4)."""
    rng = np.random.default_rng(22)
    K = 12
    frames, spacing, origin, y, w = _random_problem(rng, dims, K)
    h = float(np.prod(spacing))
    fd = _frames_dev(frames, dims, spacing, origin, torch.float32)
    whole = srb.FieldObjective(fd, list(range(K)), w, h, feature=feature, ngf_eps=0.2)
    yt = torch.as_tensor(y, dtype=torch.float32, device=fd.data.device).contiguous()
    stats, g = whole.evaluate(yt)
    N = int(np.prod(dims))
    row = dims[0]
    cuts = [0, 7 * row, 16 * row, N]
    raws, plans = [], []
    for lo, hi in zip(cuts[:-1], cuts[1:]):
        plan = srb.EvalPlan(fd, list(range(K)), feature=feature, ngf_eps=0.2, pix_range=(lo, hi))
        prob = plan.problem(y=yt)
        raws.append(plan.corr_partial(prob).clone())
        plans.append((plan, prob, lo, hi))
    total = sum(raws)
    ext = torch.stack([r[K * K + K:K * K + 3 * K] for r in raws]).amax(0)
    total[K * K + K:K * K + 3 * K] = ext
    assert int(total[-1].item()) == N
    gs = torch.zeros_like(yt)
    eng = fd.engine
    if reuse:  # the per-rank flow of parallel.py: pass 1 of the slab, then pass 2 streams its samples
        eng.set_sample_reuse(True)
    try:
        for plan, prob, lo, hi in plans:
            if reuse:
                plan.corr_partial(prob)  # this slab's samples in the engine's buffers
            plan.raw.copy_(total)
            plan.finalize(prob, w, h, n_total=N)
            assert float(plan.stats[0].item()) == pytest.approx(float(stats[0].item()), rel=1e-4)
            out = torch.empty((K, 2, hi - lo), dtype=yt.dtype, device=yt.device)
            plan.grad(prob, out, g_off=lo)
            gs[:, :, lo:hi] = out
    finally:
        eng.set_sample_reuse(False)
    assert _relmax(gs.double().cpu().numpy(), g.double().cpu().numpy()) < 1e-4


def test_deterministic_bitwise():
    rng = np.random.default_rng(5)
    frames, spacing, origin, y, w = _random_problem(rng, (64, 48), 10)
    fd = _frames_dev(frames, (64, 48), spacing, origin, torch.float32)
    obj = srb.FieldObjective(fd, list(range(10)), w)
    yt = torch.as_tensor(y, dtype=torch.float32, device=fd.data.device).contiguous()
    s1, g1 = obj.evaluate(yt)
    s1, g1 = s1.clone(), g1.clone()
    s2, g2 = obj.evaluate(yt)
    assert torch.equal(s1, s2) and torch.equal(g1, g2)


@pytest.mark.parametrize("feature", ["ncc", "ngf"])
def test_graph_replay_matches_eager(feature):
    """sr_evaluate captures a repeated evaluation as a CUDA graph (2nd call) and replays it (3rd+):
    bitwise the eager result on the same y, and the oracle's after y is rewritten in place."""
    rng = np.random.default_rng(11)
    dims, K = (40, 36), 24
    frames, spacing, origin, y, w = _random_problem(rng, dims, K)
    fd = _frames_dev(frames, dims, spacing, origin, torch.float32)
    h = float(np.prod(spacing))
    obj = srb.FieldObjective(fd, list(range(K)), w, h, feature=feature, ngf_eps=0.2)
    yt = torch.as_tensor(y, dtype=torch.float32, device=fd.data.device).contiguous()
    g = torch.empty_like(yt)
    outs = []
    for _ in range(3):  # eager, capture + launch, replay
        s, _ = obj.evaluate(yt, g)
        outs.append((s.clone(), g.clone()))
    for s, gg in outs[1:]:
        assert torch.equal(s[:4], outs[0][0][:4]) and torch.equal(gg, outs[0][1])
    y2 = y + 0.1 * rng.standard_normal(y.shape) * np.asarray(spacing)[None, :, None]
    yt.copy_(torch.as_tensor(y2, dtype=torch.float32))
    s, _ = obj.evaluate(yt, g)  # replay on new contents
    q = frames.astype(np.float32).astype(np.float64)
    yq = yt.double().cpu().numpy()
    _, Dref, gref = orc.evaluate_field(list(q), dims, spacing, origin, yq, w, h, feature, 0.2)
    assert float(s[0].item()) == pytest.approx(Dref, rel=1e-4)
    assert _relmax(g.double().cpu().numpy(), gref) < 1e-4


def test_degenerate_and_outside_fields():
    """A frame warped entirely outside the hull is constant (0): degenerate, zero C row and
    zero gradient, exactly like the reference's zero feature vector (similarity.py:84-86)."""
    rng = np.random.default_rng(6)
    dims, K = (20, 16), 4
    frames, spacing, origin, y, w = _random_problem(rng, dims, K)
    y[2] += 1000.0
    fd = _frames_dev(frames, dims, spacing, origin, torch.float64)
    obj = srb.FieldObjective(fd, list(range(K)), w, 1.0)
    stats, g = obj.evaluate(torch.as_tensor(y, device=fd.data.device).contiguous())
    hs = obj.host_stats()
    assert hs["degenerate"].tolist() == [False, False, True, False]
    assert np.all(hs["corr"][2] == 0) and np.all(hs["corr"][:, 2] == 0)
    assert torch.all(g[2] == 0)
    st, Dref, gref = orc.evaluate_field([frames[k] for k in range(K)], dims, spacing, origin, y, w, 1.0)
    assert float(stats[0].item()) == pytest.approx(Dref, rel=1e-10)
    assert _relmax(g.cpu().numpy(), gref) < 1e-10


def test_single_frame_and_bad_args():
    rng = np.random.default_rng(7)
    frames, spacing, origin, y, w = _random_problem(rng, (8, 8), 1)
    fd = _frames_dev(frames, (8, 8), spacing, origin, torch.float64)
    obj = srb.FieldObjective(fd, [0], w, 1.0)
    stats, g = obj.evaluate(torch.as_tensor(y, device=fd.data.device).contiguous())
    # one frame: C = [[1]], the projected direction vanishes (the reference leaves ~1e-17)
    assert float(stats[0].item()) == 0.0 and float(g.abs().max()) < 1e-12
    with pytest.raises(ValueError):
        srb.FieldObjective(fd, [0], [1.0, 2.0], 1.0)
    with pytest.raises(NotImplementedError):
        srb.FieldObjective(fd, [0] * 161, np.ones(161), 1.0).evaluate(  # > SR_MAX_FRAMES = 160
            torch.zeros((161, 2, 64), dtype=torch.float64, device=fd.data.device))


@pytest.mark.parametrize("dims", [(40, 24), (12, 10, 9)])
def test_curvature_fused_ngf_pass2(dims):
    """sr_evaluate_reg on the split fp32 NGF path adds alpha h L L (y - x) inside k_ngf_adj4: the gradient is
    the unfused one (sr_evaluate then sr_curvature) up to the contraction of the final addition (1 ulp of a
    few entries: 1e-6 of max |g|) and S agrees to 1e-12;
    both match the oracle (D + S and dD/dy + dS/dy) at the fp32 tolerance."""
    rng = np.random.default_rng(5)
    frames, spacing, origin, y, w = _random_problem(rng, dims, 5, amp=0.3)
    h = float(np.prod(spacing))
    fd = _frames_dev(frames, dims, spacing, origin, torch.float32)
    yt = torch.as_tensor(y).to(device=fd.data.device, dtype=torch.float32).contiguous()
    obj = srb.FieldObjective(fd, list(range(5)), w, h, feature="ngf", ngf_eps=0.5, alpha=1.5)
    stats, g = obj.evaluate(yt)
    S = float(obj.s_reg.item())
    D = float(stats[0].item())
    plan = obj.plan
    prob = plan.problem(y=yt)
    g2 = torch.empty_like(yt)
    s2 = torch.zeros(1, dtype=torch.float64, device=yt.device)
    plan.evaluate(prob, w, h, g2)
    plan.curvature(prob, 1.5, h, g2, s2)
    assert float((g - g2).abs().max()) <= 1e-6 * float(g.abs().max())
    assert S == pytest.approx(float(s2.item()), rel=1e-12)
    q = frames.astype(np.float32).astype(np.float64)
    yq = y.astype(np.float32).astype(np.float64)
    _, Dref, gref = orc.evaluate_field(list(q), dims, spacing, origin, yq, w, h, "ngf", 0.5)
    Sref, gS = orc.curvature(yq, dims, spacing, origin, 1.5, h)
    assert D == pytest.approx(Dref, rel=1e-4)
    assert S == pytest.approx(Sref, rel=1e-4)
    assert _relmax(g.double().cpu().numpy(), gref + gS) < 1e-4


@pytest.mark.parametrize("name", ["aff2d_small_0", "aff2d_subset_outside", "aff3d_small", "aff2d_degenerate"])
def test_lazy_features_match_reference(name, golden):
    """CorrelationState.features (similarity.py:109-125) materialised on first access from the device's warped
    values: equal to the reference's own feature matrix (run here from baseline/_ref) to 1e-12, zero columns for
    degenerate frames, and features^T features == corr."""
    from seqreg import similarity as ref_sim

    case = golden[name]
    seq, stack, subset = _seq_stack(case)
    st = srb.correlation_state(seq, stack, subset, case["weights"], float(case["h"]))
    ref = ref_sim.correlation_state(seq, stack, subset, case["weights"], float(case["h"]))
    f = st.features
    assert f.shape == ref.features.shape
    np.testing.assert_allclose(f, ref.features, rtol=0, atol=1e-12)
    np.testing.assert_allclose(f.T @ f, st.corr, rtol=0, atol=1e-12)
    assert st.features is f  # materialised once


def test_context_orders_calls_across_streams():
    """Evaluations issued on alternating torch streams against one context (shared scratch) give the
    same D and gradient as on one stream: sr_set_stream makes the new stream wait for the old one."""
    rng = np.random.default_rng(9)
    dims = (96, 80)
    frames, spacing, origin, y, w = _random_problem(rng, dims, 12, amp=0.3)
    fd = _frames_dev(frames, dims, spacing, origin, torch.float32)
    obj = srb.FieldObjective(fd, list(range(12)), w, float(np.prod(spacing)))
    yt = torch.as_tensor(y).to(device=fd.data.device, dtype=torch.float32).contiguous()
    stats, g = obj.evaluate(yt)
    D0, g0 = float(stats[0].item()), g.clone()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i in range(6):
        with torch.cuda.stream(streams[i % 2]):
            st, gi = obj.evaluate(yt, torch.empty_like(yt))
            outs.append((st[0].clone(), gi))
    torch.cuda.synchronize()
    for d, gi in outs:
        assert float(d.item()) == D0
        assert torch.equal(gi, g0)


@pytest.mark.parametrize("sp", [(0.5, 0.25), (0.3, 0.7)])  # power-of-two and general spacings (POW2 template)
@pytest.mark.parametrize("dims,K", [((62, 5), 3), ((64, 2), 4), ((126, 9), 5), ((130, 40), 40), ((2, 7), 3),
                                    ((1024, 3), 2), ((190, 70), 70), ((2048, 6), 2)])
def test_ngf_fast_sampler_matches_generic(dims, K, sp):
    """k_ngf_sfeat2f (one warp per 62-column chunk and row segment, shuffles, rsqrt.approx) against the generic
    k_ngf_sfeat2 (SEQREG_B200_SFEAT=0, read at launch) on ragged shapes: a single chunk, a chunk of 2 columns,
    2- and 3-row images (every look-ahead row missing), several segments, K in each Gram bucket.  Same D to
    1e-6 and the same gradient to 1e-5 of its max (rsqrt.approx is 2^-22 relative), and both match the oracle
    at the fp32 tolerance."""
    import os

    rng = np.random.default_rng(11)
    org = (-3.0, 1.0)
    from scipy.ndimage import gaussian_filter

    frames = np.stack([gaussian_filter(rng.standard_normal(dims), 1.2, mode="reflect").ravel(order="F") + 2.0
                       for _ in range(K)])
    x = orc.cell_centers(dims, sp, org).T
    y = x[None] + 0.35 * rng.standard_normal((K,) + x.shape) * np.asarray(sp)[None, :, None]
    t_ = (y - np.asarray(org)[None, :, None]) / np.asarray(sp)[None, :, None] - 0.5
    fr = t_ - np.floor(t_)
    y = np.where((fr < 2e-3) | (fr > 1 - 2e-3), y + 5e-3 * np.asarray(sp)[None, :, None], y)
    w = rng.uniform(0.5, 1.0, K)
    h = float(np.prod(sp))
    fd = _frames_dev(frames, dims, sp, org, torch.float32)
    res = []
    old = os.environ.get("SEQREG_B200_SFEAT")
    try:
        for flag in (None, "0"):
            if flag is None:
                os.environ.pop("SEQREG_B200_SFEAT", None)
            else:
                os.environ["SEQREG_B200_SFEAT"] = flag
            obj = srb.FieldObjective(fd, list(range(K)), w, h, feature="ngf", ngf_eps=0.3)
            yt = torch.as_tensor(y).to(device=fd.data.device, dtype=torch.float32).contiguous()
            stats, g = obj.evaluate(yt)  # a fresh objective and iterate: the eager path, no graph replay
            res.append((float(stats[0].item()), g.double().cpu().numpy().copy()))
    finally:
        if old is None:
            os.environ.pop("SEQREG_B200_SFEAT", None)
        else:
            os.environ["SEQREG_B200_SFEAT"] = old
    (Df, gf), (Dg, gg) = res
    assert Df == pytest.approx(Dg, rel=1e-6)
    assert np.abs(gf - gg).max() <= 1e-5 * np.abs(gg).max()
    q = frames.astype(np.float32).astype(np.float64)
    yq = y.astype(np.float32).astype(np.float64)
    _, Dref, gref = orc.evaluate_field(list(q), dims, sp, org, yq, w, h, "ngf", 0.3)
    assert Df == pytest.approx(Dref, rel=1e-4)
    # 2048 cells of a general spacing: the fp32 coordinate (p - o) / s itself resolves 2048 * 6e-8 = 1.2e-4 cells,
    # so the fractions (and the gradient of the bilinear interpolant) of both samplers carry that
    tol = 1e-4 if dims[0] <= 1024 else 5e-4
    assert _relmax(gf, gref) < tol
