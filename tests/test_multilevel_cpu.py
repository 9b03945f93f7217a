"""Host logic of the multilevel displacement-field driver (paper_2001_06613_b200/multilevel.py) and its CPU
checker (oracle.seqreg_oracle.field_stml_run): the temporal schedule and quadrature weights equal the
reference's (temporal.py:87-106, similarity.py:42-70), and the oracle driver's composition runs end to end
on a small sequence (every solve logged, fields on the finest grid)."""

import numpy as np
import pytest

from oracle import seqreg_oracle as orc
from paper_2001_06613_b200 import multilevel as ml
from paper_2001_06613_b200 import synth


@pytest.mark.parametrize("n,c", [(10, 4), (10, 3), (64, 9), (129, 17), (17, 3), (5, 5), (3, 3)])
def test_temporal_levels_match_reference(n, c):
    from seqreg.temporal import build_temporal_levels

    ref = build_temporal_levels(n, c).levels
    got = ml.temporal_levels(n, c)
    assert [tuple(k + 1 for k in lv) for lv in got] == [tuple(lv) for lv in ref]
    assert orc.temporal_levels(n, c) == got


def test_quad_weights_match_reference():
    from seqreg.similarity import default_time_interval, quad_weights

    t = np.sort(np.random.default_rng(3).uniform(0, 1, 9))
    a, b = default_time_interval(t)
    assert ml.default_time_interval(t) == (a, b)
    for sub in ([0, 3, 8], list(range(9)), [2, 5]):
        np.testing.assert_array_equal(ml.quad_weights(t[sub], a, b), quad_weights(t[sub], a, b))


def test_config_validation():
    with pytest.raises(ValueError):
        ml.FieldRunConfig(spatial_levels=0)
    with pytest.raises(ValueError):
        ml.FieldRunConfig(weights="equal")
    with pytest.raises(ValueError):
        ml.FieldRunConfig(eps=0.0)


def test_oracle_driver_runs_small():
    cfg = synth.CONFIGS["c1"]
    fr, times, sp, org = synth.make_sequence(cfg, seed=0, device="cpu", K=5, dims=(16, 16))
    y, runs = orc.field_stml_run(list(fr.numpy()), (16, 16), sp, org, times, spatial_levels=2,
                                 temporal_coarsest_size=3, feature="ngf", ngf_eps=0.1, alpha=0.0,
                                 weights="uniform", eps=None,
                                 optim=dict(max_iters=3, grad_tol=1e-30, f_tol=1e-30, step_tol=1e-30))
    assert y.shape == (5, 2, 256)
    assert [(r["spatial_level"], r["temporal_level"]) for r in runs] == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert all(np.isfinite(r["f_final"]) and r["f_final"] <= r["f_initial"] for r in runs)
