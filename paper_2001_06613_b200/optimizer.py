"""Device-resident L-BFGS: mirror of ``seqreg.optimizer`` (/root/reference/pkg/src/seqreg/optimizer.py).

Same names, option defaults, validation messages, result fields and stop reasons as the
reference; the iterate, the gradient, the search direction and the curvature history live in
device memory (fp64) and the vector algebra runs in ``csrc/lbfgs.cu`` (``sr_lbfgs_minimize``).

Two calling modes, chosen by ``x0``:

* host mode (``x0`` a numpy array / sequence): ``objective(x: np.ndarray) -> ObjectiveEval`` with a
  numpy gradient, exactly the reference's contract, so the reference drivers can call it;
* device mode (``x0`` a CUDA ``torch.Tensor``): ``objective`` receives a fp64 CUDA tensor (a view
  of the driver's buffer, valid during the call) and may return a CUDA tensor gradient; nothing
  crosses PCIe except the scalars that steer the line search.

``OptimResult.x_final`` has the type of ``x0`` (numpy in host mode, a CUDA tensor in device mode).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .engine import get_engine

__all__ = ["ObjectiveEval", "OptimOptions", "OptimResult", "lbfgs_minimize", "REASONS"]

REASONS = ("grad_tol", "step_tol", "f_tol", "max_iters", "line_search_failure")


@dataclass
class ObjectiveEval:
    """Value and gradient of one objective evaluation (optimizer.py:19-24)."""

    value: float
    gradient: object


@dataclass(frozen=True)
class OptimOptions:
    """optimizer.py:27-46 (same defaults and messages)."""

    memory: int = 5
    max_iters: int = 50
    grad_tol: float = 1e-4
    step_tol: float = 1e-7
    f_tol: float = 1e-5
    armijo_c1: float = 1e-4
    backtrack_factor: float = 0.5
    max_backtracks: int = 20

    def __post_init__(self):
        if self.memory < 1 or self.max_iters < 1 or self.max_backtracks < 1:
            raise ValueError("memory, max_iters, max_backtracks must be >= 1")
        if self.grad_tol <= 0 or self.step_tol <= 0 or self.f_tol <= 0:
            raise ValueError("tolerances must be > 0")
        if not 0 < self.armijo_c1 < 1:
            raise ValueError("armijo_c1 must be in (0, 1)")
        if not 0 < self.backtrack_factor < 1:
            raise ValueError("backtrack_factor must be in (0, 1)")

    def c_struct(self) -> _lib.SrLbfgsOptions:
        return _c_options(self)


def _c_options(o) -> _lib.SrLbfgsOptions:
    """Any options object with the OptimOptions fields (ours or the reference's own)."""
    return _lib.SrLbfgsOptions(int(o.memory), int(o.max_iters), float(o.grad_tol), float(o.step_tol),
                               float(o.f_tol), float(o.armijo_c1), float(o.backtrack_factor), int(o.max_backtracks))


@dataclass
class OptimResult:
    """optimizer.py:49-56."""

    x_final: object
    f_final: float
    f_initial: float
    iterations: int
    objective_evaluations: int
    converged_reason: str  # grad_tol | step_tol | f_tol | max_iters | line_search_failure


class _DevPtr:
    """A raw fp64 device buffer of the driver, exposed to torch without a copy."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 2}


def _device_view(ptr: int, n: int, device: torch.device) -> torch.Tensor:
    return torch.as_tensor(_DevPtr(ptr, n), device=device)


def lbfgs_minimize(objective, x0, opts: OptimOptions | None = None, trace=None, *, engine=None) -> OptimResult:
    """Minimize ``x -> ObjectiveEval`` from ``x0`` (optimizer.py:76-168) with device-resident vectors.

    Stop rules, the two-loop recursion, Armijo backtracking and the curvature-pair test are the
    reference's; ``trace(iteration, f, grad_inf, step, evaluations)`` is called after each
    accepted step.  A non-finite objective at the start raises ``ValueError`` like the reference;
    an exception raised by ``objective`` or ``trace`` propagates unchanged.
    """
    if opts is None:
        opts = OptimOptions()
    elif not isinstance(opts, OptimOptions):  # e.g. the reference's own OptimOptions: same fields, same checks
        opts = OptimOptions(*(getattr(opts, f) for f in ("memory", "max_iters", "grad_tol", "step_tol", "f_tol",
                                                          "armijo_c1", "backtrack_factor", "max_backtracks")))
    eng = engine if engine is not None else get_engine()
    dev = eng.device
    device_mode = isinstance(x0, torch.Tensor) and x0.is_cuda
    x_t = torch.as_tensor(x0, dtype=torch.float64).detach().reshape(-1).to(dev).clone().contiguous()
    n = int(x_t.numel())
    if n < 1:
        raise ValueError("x0 must have at least one entry")
    errors: list[BaseException] = []

    def _objective(user, x_ptr, f_out, g_ptr):
        try:
            xv = _device_view(x_ptr, n, dev)
            if device_mode and hasattr(objective, "evaluate_into"):
                # device objectives may write the fp64 gradient straight into the solver's buffer (no
                # intermediate copies of n-vectors): evaluate_into(x, g_out) -> value
                value = objective.evaluate_into(xv, _device_view(g_ptr, n, dev))
                torch.cuda.synchronize(dev)
                f_out[0] = float(value)
                return 0
            arg = xv if device_mode else xv.cpu().numpy()
            e = objective(arg)
            g = e.gradient
            g = g.detach() if isinstance(g, torch.Tensor) else torch.as_tensor(np.asarray(g, dtype=np.float64))
            g = g.to(device=dev, dtype=torch.float64).reshape(-1)
            if g.numel() != n:
                raise ValueError(f"gradient has {g.numel()} entries, expected {n}")
            _device_view(g_ptr, n, dev).copy_(g)
            torch.cuda.synchronize(dev)
            f_out[0] = float(e.value)
            return 0
        except BaseException as exc:  # re-raised after the C call returns
            errors.append(exc)
            return 1

    def _trace(user, iteration, f, g_inf, step, evals):
        if errors:
            return
        try:
            trace(int(iteration), float(f), float(g_inf), float(step), int(evals))
        except BaseException as exc:
            errors.append(exc)

    ocb = _lib.OBJECTIVE_FN(_objective)
    tcb = _lib.TRACE_FN(_trace) if trace is not None else _lib.TRACE_FN()
    res = _lib.SrLbfgsResult()
    torch.cuda.synchronize(dev)
    status = eng.lib.sr_lbfgs_minimize(eng.ctx, n, ctypes.c_void_p(x_t.data_ptr()), ctypes.byref(_c_options(opts)),
                                       ocb, None, tcb, None, ctypes.byref(res))
    if errors:
        raise errors[0]
    _lib.check(status)
    if device_mode:
        x_final = x_t.reshape(x0.shape)
    else:
        x_final = x_t.cpu().numpy()
    return OptimResult(x_final, float(res.f_final), float(res.f_initial), int(res.iterations),
                       int(res.objective_evaluations), REASONS[res.converged_reason])
