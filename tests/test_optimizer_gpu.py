"""GPU: the device-resident L-BFGS (csrc/lbfgs.cu through sr_lbfgs_minimize) against the
reference optimizer's recorded outcomes (tests/golden/lbfgs_golden.json) and the oracle.

Vectors live in HBM and dot products use a fixed-order reduction, so x and f agree with the
reference to rounding; iteration counts, evaluation counts, stop reasons and the trace's
iteration/evaluation sequence must match exactly."""

import ctypes
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2001_06613_b200 as srb
from oracle import seqreg_oracle as orc
from paper_2001_06613_b200 import _lib
from paper_2001_06613_b200.optimizer import ObjectiveEval, OptimOptions, lbfgs_minimize
from tests.lbfgs_problems import problems

pytestmark = pytest.mark.gpu

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "lbfgs_golden.json").read_text())


def _check(res, gold, trace):
    assert (res.iterations, res.objective_evaluations, res.converged_reason) == (
        gold["iterations"], gold["objective_evaluations"], gold["converged_reason"])
    assert res.f_final == pytest.approx(gold["f_final"], rel=1e-10, abs=1e-13)
    x = res.x_final.double().cpu().numpy() if isinstance(res.x_final, torch.Tensor) else res.x_final
    xg = np.asarray(gold["x_final"])
    assert np.abs(x - xg).max() <= 1e-8 * max(1.0, np.abs(xg).max())
    assert [(int(t[0]), int(t[4])) for t in trace] == [(int(t[0]), int(t[4])) for t in gold["trace"]]


@pytest.mark.parametrize("name", sorted(GOLDEN))
def test_device_lbfgs_host_mode_matches_reference(name):
    fn, x0, opts = problems()[name]
    trace = []
    res = lbfgs_minimize(lambda x: ObjectiveEval(*fn(x)), x0, OptimOptions(**opts),
                         trace=lambda *a: trace.append(a))
    assert isinstance(res.x_final, np.ndarray)
    _check(res, GOLDEN[name], trace)


@pytest.mark.parametrize("name", ["quadratic", "rosenbrock", "logcosh"])
def test_device_lbfgs_device_mode(name):
    """Objective on CUDA tensors: the iterate never leaves the device."""
    fn, x0, opts = problems()[name]

    def obj(x):  # torch restatement of the numpy problem on the device
        assert x.is_cuda and x.dtype == torch.float64
        f, g = fn(x.cpu().numpy())
        return ObjectiveEval(f, torch.as_tensor(g, device=x.device))

    trace = []
    res = lbfgs_minimize(obj, torch.as_tensor(x0, device="cuda"), OptimOptions(**opts),
                         trace=lambda *a: trace.append(a))
    assert isinstance(res.x_final, torch.Tensor) and res.x_final.is_cuda
    _check(res, GOLDEN[name], trace)


def test_nonfinite_start_and_callback_errors():
    with pytest.raises(ValueError, match="not finite at the starting point"):
        lbfgs_minimize(lambda x: ObjectiveEval(float("nan"), np.zeros_like(x)), np.zeros(4))

    class Boom(RuntimeError):
        pass

    def bad(x):
        raise Boom("from the objective")

    with pytest.raises(Boom):
        lbfgs_minimize(bad, np.zeros(4))
    with pytest.raises(ValueError, match="expected 4"):
        lbfgs_minimize(lambda x: ObjectiveEval(1.0, np.zeros(3)), np.zeros(4))


def test_c_abi_validates_options():
    eng = srb.get_engine()
    o = _lib.SrLbfgsOptions()
    eng.lib.sr_lbfgs_defaults(ctypes.byref(o))
    assert (o.memory, o.max_iters, o.max_backtracks) == (5, 50, 20)
    o.armijo_c1 = 1.5
    x = torch.zeros(3, dtype=torch.float64, device=eng.device)
    res = _lib.SrLbfgsResult()
    cb = _lib.OBJECTIVE_FN(lambda u, xp, f, gp: 0)
    st = eng.lib.sr_lbfgs_minimize(eng.ctx, 3, ctypes.c_void_p(x.data_ptr()), ctypes.byref(o), cb, None,
                                   _lib.TRACE_FN(), None, ctypes.byref(res))
    with pytest.raises(ValueError, match=r"armijo_c1 must be in \(0, 1\)"):
        _lib.check(st)


def test_registration_objective_device_vs_oracle_lbfgs():
    """D(y) of a displacement field (fp64 engine, perturbed start) minimised by the device L-BFGS in
    device mode and by the oracle L-BFGS on the same objective: same iterations, evaluations and
    stop reason, D decreasing."""
    from paper_2001_06613_b200 import synth

    cfg = synth.CONFIGS["c1"]
    dims, K = (64, 64), 6
    frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device="cuda", K=K, dims=dims)
    fd = srb.DeviceFrames(srb.get_engine(), frames.to(torch.float64), srb.GridSpec(dims, spacing, origin))
    h = float(np.prod(spacing))
    obj = srb.FieldObjective(fd, list(range(K)), np.full(K, 1.0 / K), h)
    x0 = synth.smooth_noise_iterate(dims, K, sigma_px=3.0, std_px=0.5, device="cuda").to(torch.float64).contiguous()

    def dev_obj(x):
        y = x.reshape(x0.shape).contiguous()
        stats, g = obj.evaluate(y)
        return ObjectiveEval(float(stats[0].item()), g.reshape(-1).double())

    opts = dict(max_iters=12, grad_tol=1e-12, f_tol=1e-14, step_tol=1e-14)
    res = lbfgs_minimize(dev_obj, x0.double(), OptimOptions(**opts))

    def host_obj(x):
        e = dev_obj(torch.as_tensor(x, device="cuda"))
        return e.value, e.gradient.cpu().numpy()

    ref = orc.lbfgs_minimize(host_obj, x0.double().reshape(-1).cpu().numpy(), **opts)
    assert (res.iterations, res.objective_evaluations, res.converged_reason) == (
        ref["iterations"], ref["objective_evaluations"], ref["converged_reason"])
    assert res.f_final == pytest.approx(ref["f_final"], rel=1e-9)
    assert res.f_final < res.f_initial
