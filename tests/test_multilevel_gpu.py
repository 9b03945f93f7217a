"""BASELINE C1 end to end on the device: the spatio-temporal multilevel displacement-field run
(paper_2001_06613_b200.multilevel.field_stml_run: build_pyramid, device L-BFGS on FieldObjective with NGF
and curvature, interp_linear_fields / ls_predict_fields between temporal levels, prolong_field between
spatial levels; control flow temporal.py:376-457) against the same composition on the CPU oracle
(oracle.seqreg_oracle.field_stml_run / field_solve), fp64.

C1: K = 10, 128^2, 3 spatial levels (32/64/128), temporal levels {every 4th, 2nd, all} (coarsest size 4),
NGF eps 0.1, curvature alpha = 1, w_i = 1/K, 20 iterations per level (tolerances 1e-30), every level run.

Two checks (tolerances written here):
  * per solve, from the same starting fields: the oracle's L-BFGS replay of each of the 9 solves gives the
    identical iteration count, evaluation count and stop reason, f within 1e-10 of f_initial and the final
    fields within 1e-10 of the largest displacement (north_star fp64 tolerance).  (Without the regulariser,
    alpha = 0, not a BASELINE config, the problem is ill-conditioned: measured, 20 L-BFGS iterations amplify
    the 1e-16 differences to ~2e-9 in f and ~1e-6 in the fields, with identical iteration and evaluation
    counts; it is not asserted here.)
  * the whole chained run: identical iteration counts at every level (north_star), the final all-frames
    dissimilarity within 1e-6 relative and the final fields within 1e-6 of the largest displacement.  Chained
    over 9 solves of 20 L-BFGS iterations, the 1e-16 rounding differences of reductions are amplified by
    the optimiser (and an Armijo test can land on the other side), so the chained run is held to 1e-6, each
    solve to 1e-10."""

import numpy as np
import pytest
import torch

from oracle import seqreg_oracle as orc
import paper_2001_06613_b200 as srb
from paper_2001_06613_b200 import multilevel as ml
from paper_2001_06613_b200 import synth
from paper_2001_06613_b200.optimizer import OptimOptions

pytestmark = pytest.mark.gpu

ITERS = dict(max_iters=20, grad_tol=1e-30, f_tol=1e-30, step_tol=1e-30)


def _c1():
    cfg = synth.CONFIGS["c1"]
    fr, times, sp, org = synth.make_sequence(cfg, seed=0, device="cpu")
    return cfg, fr.numpy(), times, sp, org


@pytest.fixture(scope="module")
def c1_run():
    alpha = 1.0
    cfg, fr, times, sp, org = _c1()
    fcfg = ml.FieldRunConfig(spatial_levels=3, temporal_coarsest_size=4, feature="ngf", ngf_eps=0.1, alpha=alpha,
                             weights="uniform", eps=None, optim=OptimOptions(**ITERS))
    eng = srb.get_engine(0)
    fd = srb.DeviceFrames.from_array(eng, fr, srb.GridSpec(cfg.dims, sp, org), torch.float64)
    y, runs = ml.field_stml_run(fd, times, fcfg, keep_fields=True)
    torch.cuda.synchronize()
    return alpha, cfg, fr, times, sp, org, y, runs


def test_c1_each_solve_matches_oracle(c1_run):
    alpha, cfg, fr, times, sp, org, y, runs = c1_run
    tol = tol_y = 1e-10
    pyr = orc.field_pyramid(list(fr), cfg.dims, sp, 3)
    assert len(runs) == 9
    for r in runs:
        lf, dm, lsp = pyr[r.spatial_level]
        h = float(np.prod(lsp))
        w = np.full(len(r.active), 1.0 / len(fr))
        y0 = r.y_init.cpu().numpy()
        y1, q = orc.field_solve([lf[k] for k in r.active], dm, lsp, org, y0, w, h, "ngf", 0.1, alpha, ITERS, 8, True)
        assert (r.iterations, r.evaluations, r.reason) == (q["iterations"], q["objective_evaluations"],
                                                           q["converged_reason"]), (r.spatial_level, r.temporal_level)
        fscale = abs(q["f_initial"])
        assert abs(r.f_initial - q["f_initial"]) <= 1e-10 * fscale
        assert abs(r.f_final - q["f_final"]) <= tol * fscale
        x = orc.cell_centers(dm, lsp, org).T
        dscale = max(np.abs(y1 - x[None]).max(), lsp[0])
        err = np.abs(r.y_final.cpu().numpy() - y1).max() / dscale
        assert err <= tol_y, (r.spatial_level, r.temporal_level, err)


def test_c1_chained_run_matches_oracle(c1_run):
    alpha, cfg, fr, times, sp, org, y, runs = c1_run
    y_ref, runs_ref = orc.field_stml_run(list(fr), cfg.dims, sp, org, times, 3, 4, "ngf", 0.1, alpha, "uniform",
                                         1e-5, None, ITERS, threads=8)
    assert [r.iterations for r in runs] == [q["iterations"] for q in runs_ref]
    d, dr = runs[-1].dissim_all, runs_ref[-1]["dissim_all"]
    assert abs(d - dr) <= 1e-6 * abs(dr)
    x = orc.cell_centers(cfg.dims, sp, org).T
    dscale = max(np.abs(y_ref - x[None]).max(), sp[0])
    assert np.abs(y.cpu().numpy() - y_ref).max() <= 1e-6 * dscale
    print(f"alpha={alpha}: runs", [(r.iterations, r.evaluations, r.reason) for r in runs],
          "oracle", [(q["iterations"], q["evaluations"], q["reason"]) for q in runs_ref])
