"""Generate golden vectors by running the REFERENCE implementation (seqreg) here.

Run in the build container (where /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Each case stores its inputs (or the seed that
regenerates them through paper_2001_06613_b200.synth) and the reference outputs of
  correlation_state / dissimilarity / dissimilarity_gradient   (similarity.py:128-220)
  ls_predict / _interp_linear / thomas_solve                   (temporal.py:109-239)
The GPU box has no /root/reference: tests compare against these files.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, "/root/reference/pkg/src")

from scipy.ndimage import gaussian_filter  # noqa: E402

import seqreg  # noqa: E402
from seqreg import (  # noqa: E402
    Affine,
    AffineStack,
    Grid,
    Image,
    ImageSequence,
    correlation_state,
    dissimilarity,
    dissimilarity_gradient,
)
from seqreg.temporal import _interp_linear, ls_predict  # noqa: E402

from paper_2001_06613_b200 import synth  # noqa: E402

CASES = {}


def add_affine_case(name, seq, rows, subset, weights, h, store_frames=True, extra=None):
    d = seq.grid.ndim
    stack = AffineStack.from_params(rows, subset, seq.frame_count, d)
    st = correlation_state(seq, stack, subset, weights, h)
    D = dissimilarity(st)
    g = dissimilarity_gradient(st, seq, stack, subset)
    case = {
        "dims": np.array(seq.grid.dims),
        "spacing": np.array(seq.grid.spacing),
        "origin": np.array(seq.grid.origin),
        "times": np.array(seq.times),
        "rows": np.asarray(rows, dtype=np.float64),
        "subset": np.array(subset),
        "weights": np.asarray(weights, dtype=np.float64),
        "h": np.array(h),
        "corr": st.corr,
        "D": np.array(D),
        "grad": g,
        "degenerate": st.degenerate,
        "center_norms": st.center_norms,
    }
    if store_frames:
        case["frames"] = np.stack([f.values for f in seq.frames])
    if extra:
        case.update(extra)
    CASES[name] = case


def smooth_seq(rng, dims, n, spacing=None, origin=None):
    spacing = spacing or (1.0,) * len(dims)
    origin = origin or tuple(-d / 2 for d in dims)
    grid = Grid(dims, spacing, origin)
    frames = [Image(grid, gaussian_filter(rng.standard_normal(dims), 1.5, mode="reflect").ravel(order="F"))
              for _ in range(n)]
    return ImageSequence(frames, list(range(n)))


def ident_rows(d, n):
    return np.tile(np.concatenate([np.eye(d).ravel(), np.zeros(d)]), (n, 1))


def main():
    rng = np.random.default_rng(1234)
    # 1. the test_similarity FD setting: 8x8, 3 frames, perturbed affines
    for i in range(3):
        seq = smooth_seq(rng, (8, 8), 3)
        rows = ident_rows(2, 3) + 0.02 * rng.standard_normal((3, 6))
        a, b = seqreg.default_time_interval(seq.times)
        w = seqreg.quad_weights(seq.times, a, b)
        add_affine_case(f"aff2d_small_{i}", seq, rows, (1, 2, 3), w, seq.grid.cell_volume)
    # 2. identity start (every sample on a node: the kink case), dyadic grid
    seq = smooth_seq(rng, (16, 16), 5, spacing=(1 / 16, 1 / 16), origin=(0.0, 0.0))
    add_affine_case("aff2d_identity_dyadic", seq, ident_rows(2, 5), (1, 2, 3, 4, 5), np.full(5, 0.2),
                    seq.grid.cell_volume)
    # 3. identity on a non-dyadic grid (true division path)
    seq = smooth_seq(rng, (12, 10), 4, spacing=(0.1, 0.3), origin=(-0.7, 1.1))
    add_affine_case("aff2d_identity_nondyadic", seq, ident_rows(2, 4), (1, 2, 3, 4), np.full(4, 0.25), 0.03)
    # 4. subset of frames, rectangular grid, larger motion (some samples leave the hull)
    seq = smooth_seq(rng, (20, 14), 6, spacing=(0.5, 0.25), origin=(-5.0, -1.75))
    rows = ident_rows(2, 3) + np.array([0.03, 0.01, -0.02, 0.04, 0.9, -0.6]) * rng.standard_normal((3, 6))
    add_affine_case("aff2d_subset_outside", seq, rows, (2, 4, 6), np.array([0.3, 0.5, 0.2]), seq.grid.cell_volume)
    # 5. 3-D, non-dyadic spacing
    seq = smooth_seq(rng, (7, 6, 5), 4, spacing=(1.0, 0.8, 1.3), origin=(-3.5, -2.4, -3.25))
    rows = ident_rows(3, 4) + 0.02 * rng.standard_normal((4, 12))
    add_affine_case("aff3d_small", seq, rows, (1, 2, 3, 4), np.full(4, 0.25), seq.grid.cell_volume)
    # 6. degenerate (constant) frame -> zero corr row, zero gradient row
    grid = Grid((9, 7), (1.0, 1.0), (0.0, 0.0))
    vals = [gaussian_filter(rng.standard_normal((9, 7)), 1.2).ravel(order="F") for _ in range(2)]
    seq = ImageSequence([Image(grid, vals[0]), Image(grid, np.full(63, 2.0)), Image(grid, vals[1])], [0, 1, 2])
    add_affine_case("aff2d_degenerate", seq, ident_rows(2, 3) + 0.01 * rng.standard_normal((3, 6)),
                    (1, 2, 3), np.full(3, 1 / 3), 1.0)
    # 7. config-1 shape (128^2, K=10, fp64) on the synthetic blob sequence (regenerated from seed)
    cfg = synth.CONFIGS["c1"]
    frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device="cpu")
    frames = frames.numpy()
    grid = Grid(cfg.dims, spacing, origin)
    seq = ImageSequence([Image(grid, f) for f in frames], list(times))
    w = np.full(cfg.K, 1.0 / cfg.K)
    add_affine_case("c1_identity", seq, ident_rows(2, cfg.K), tuple(range(1, cfg.K + 1)), w,
                    grid.cell_volume, store_frames=False, extra={"synth": np.array("c1:0")})
    rows = ident_rows(2, cfg.K) + np.array([0.01, 0.01, 0.01, 0.01, 0.005, 0.005]) * rng.standard_normal((cfg.K, 6))
    add_affine_case("c1_perturbed", seq, rows, tuple(range(1, cfg.K + 1)), w, grid.cell_volume,
                    store_frames=False, extra={"synth": np.array("c1:0")})
    add_affine_case("c1_subset", seq, rows[[0, 4, 8, 9]], (1, 5, 9, 10), np.full(4, 0.25), grid.cell_volume,
                    store_frames=False, extra={"synth": np.array("c1:0")})
    # 8. temporal predictors on an affine stack (temporal.py:109-127, 194-239)
    n = 9
    times = np.sort(rng.uniform(0, 1, n))
    ref_rows = ident_rows(2, n) + 0.05 * rng.standard_normal((n, 6))
    active = (1, 3, 5, 9)
    eta_rows = ref_rows[[k - 1 for k in active]] + 0.01 * rng.standard_normal((len(active), 6))
    ref = AffineStack.from_params(ref_rows, range(1, n + 1), n, 2)
    eta = AffineStack.from_params(eta_rows, active, n, 2)
    z = ls_predict(eta, ref, 0.7, times).params_matrix()
    lin = _interp_linear(eta, active, range(1, n + 1), times).params_matrix()
    CASES["temporal"] = {"times": times, "ref": ref_rows, "active": np.array(active), "eta": eta_rows,
                         "beta": np.array(0.7), "ls": z, "interp": lin}
    out = {}
    for name, case in CASES.items():
        for key, val in case.items():
            out[f"{name}/{key}"] = val
    np.savez_compressed(HERE / "golden.npz", **out)
    print(f"wrote {len(CASES)} cases to {HERE / 'golden.npz'}")


if __name__ == "__main__":
    main()
