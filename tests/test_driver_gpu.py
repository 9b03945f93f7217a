"""The reference's own multilevel drivers (spml_run / stml_run, temporal.py:355-457) running on
the B200 engine through install(): same iteration and evaluation counts as the CPU reference at
fixed iterations, same final transforms (fp64).  Needs the reference package importable
(baseline/_ref, installed by __graft_entry__.build() from the reference sources; it travels to the
GPU box with the repo snapshot).  A missing reference FAILS these tests (it is not a skip)."""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
_REF = ROOT / "baseline" / "_ref"
if str(_REF) not in sys.path:
    sys.path.append(str(_REF))
try:
    import seqreg
except ImportError as exc:  # collected on CPU too: fail the (gpu-marked) tests, not the collection
    seqreg = None
    _SEQREG_ERR = str(exc)


@pytest.fixture(autouse=True)
def _need_reference():
    if seqreg is None:
        pytest.fail(f"reference package not importable from baseline/_ref ({_SEQREG_ERR}); run build()")

import paper_2001_06613_b200 as srb  # noqa: E402

pytestmark = pytest.mark.gpu


def _run(method, seq, cfg):
    pyr = seqreg.build_pyramid(seq, cfg.spatial_levels)
    if method == "spml":
        return seqreg.spml_run(pyr, cfg)
    sched = seqreg.build_temporal_levels(seq.frame_count, cfg.temporal_coarsest_size)
    return seqreg.stml_run(pyr, sched, cfg)


@pytest.mark.parametrize("method", ["spml", "stml"])
def test_reference_driver_on_gpu_matches_cpu(method):
    seq, truth = seqreg.synth_generate(seqreg.SynthSpec(dims=(48, 40), frames=9, seed=3))
    opts = seqreg.OptimOptions(max_iters=6, grad_tol=1e-30, step_tol=1e-30, f_tol=1e-30)
    cfg = seqreg.RunConfig(spatial_levels=2, temporal_coarsest_size=3, optim=opts)
    stack_cpu, runs_cpu = _run(method, seq, cfg)
    srb.configure(dtype=torch.float64, feature="ncc")
    srb.install()
    try:
        stack_gpu, runs_gpu = _run(method, seq, cfg)
    finally:
        srb.uninstall()
    assert len(runs_cpu) == len(runs_gpu)
    for rc, rg in zip(runs_cpu, runs_gpu):
        assert rc.result.iterations == rg.result.iterations
        assert rc.result.objective_evaluations == rg.result.objective_evaluations
        assert rc.result.converged_reason == rg.result.converged_reason
        assert rg.result.f_final == pytest.approx(rc.result.f_final, rel=1e-8)
        assert rg.dissim_all == pytest.approx(rc.dissim_all, rel=1e-8)
    a, b = stack_cpu.params_matrix(), stack_gpu.params_matrix()
    assert np.abs(a - b).max() <= 1e-8 * max(1.0, np.abs(a).max())


@pytest.mark.parametrize("method", ["spml", "stml"])
def test_reference_driver_with_device_lbfgs(method):
    """The reference drivers with both the evaluation (install()) and the optimizer
    (seqreg.temporal.lbfgs_minimize -> the device L-BFGS, host mode) replaced: same iteration /
    evaluation counts, stop reasons and final objective as the CPU reference."""
    import seqreg.temporal as T

    from paper_2001_06613_b200 import optimizer as dev_opt

    seq, truth = seqreg.synth_generate(seqreg.SynthSpec(dims=(48, 40), frames=9, seed=4))
    opts = seqreg.OptimOptions(max_iters=8, grad_tol=1e-30, step_tol=1e-30, f_tol=1e-30)
    cfg = seqreg.RunConfig(spatial_levels=2, temporal_coarsest_size=3, optim=opts)
    stack_cpu, runs_cpu = _run(method, seq, cfg)
    srb.configure(dtype=torch.float64, feature="ncc")
    srb.install()
    saved = T.lbfgs_minimize
    T.lbfgs_minimize = dev_opt.lbfgs_minimize
    try:
        stack_gpu, runs_gpu = _run(method, seq, cfg)
    finally:
        T.lbfgs_minimize = saved
        srb.uninstall()
    assert len(runs_cpu) == len(runs_gpu)
    for rc, rg in zip(runs_cpu, runs_gpu):
        assert (rc.result.iterations, rc.result.objective_evaluations, rc.result.converged_reason) == (
            rg.result.iterations, rg.result.objective_evaluations, rg.result.converged_reason)
        assert rg.result.f_final == pytest.approx(rc.result.f_final, rel=1e-8)
    a, b = stack_cpu.params_matrix(), stack_gpu.params_matrix()
    assert np.abs(a - b).max() <= 1e-7 * max(1.0, np.abs(a).max())
