"""Displacement-field objective: D(y), dD/dy (and the curvature regulariser S(y)) for
per-cell sample positions y_k(x), the north_star parametrisation.

The reference only has affine transforms (transform.py:35-96); this module is
the same objective (similarity.py:128-220) with y_k(x) free per cell.  It
reduces to the reference exactly when y_k(x) = A_k x + b_k (the
affine-contraction identity; tests/test_parity_gpu.py).

Two call paths:
  * ``evaluate(y)``          device tensors in, device tensors out (no host sync);
  * ``evaluate_host(y_np)``  the end-to-end path a host optimiser uses: pinned host
                             buffers, H2D of y, evaluation, D2H of D and dD/dy.
"""

from __future__ import annotations

import numpy as np
import torch

from .engine import DeviceFrames, EvalPlan

__all__ = ["FieldObjective"]


class FieldObjective:
    """Objective over the subset ``frame_index`` (0-based) of a device frame stack.

    Parameters mirror the reference's correlation_state(seq, stack, subset,
    weights, cell_volume): ``weights`` one per subset frame, ``cell_volume`` h
    (defaults to the grid's cell volume, grid.py:97-99).  ``alpha`` > 0 adds the
    curvature regulariser S(y) = alpha/2 h sum ||L (y - x)||^2.
    """

    def __init__(self, frames: DeviceFrames, frame_index, weights, cell_volume: float | None = None, *,
                 feature: str = "ncc", ngf_eps: float = 0.1, alpha: float = 0.0):
        self.frames = frames
        self.plan = EvalPlan(frames, frame_index, feature=feature, ngf_eps=ngf_eps)
        self.k = self.plan.k
        self.grid = frames.grid
        self.weights = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        if self.weights.size != self.k:
            raise ValueError("one weight per subset frame required")
        self.cell_volume = self.grid.cell_volume if cell_volume is None else float(cell_volume)
        self.alpha = float(alpha)
        dev = frames.data.device
        self.s_reg = torch.zeros(1, dtype=torch.float64, device=dev)
        self._pinned_y = None
        self._pinned_g = None
        self._dev_y = None
        self._dev_g = None

    @property
    def shape(self) -> tuple:
        return (self.k, self.grid.ndim, self.grid.cell_count)

    def identity(self) -> torch.Tensor:
        """y_k(x) = x for every subset frame: the cell centres (grid.py:170-187)."""
        axes = [self.grid.origin[a] + (np.arange(self.grid.dims[a]) + 0.5) * self.grid.spacing[a]
                for a in range(self.grid.ndim)]
        mesh = np.meshgrid(*axes, indexing="ij")
        x = np.stack([m.ravel(order="F") for m in mesh])
        y = np.broadcast_to(x, self.shape).copy()
        return torch.as_tensor(y).to(device=self.frames.data.device, dtype=self.frames.dtype)

    def evaluate(self, y: torch.Tensor, grad: torch.Tensor | None = None, *, want_grad: bool = True):
        """Returns the device stats buffer (D = stats[0]); fills ``grad`` with dD/dy (+ dS/dy).

        With alpha > 0, S(y) is in ``self.s_reg[0]`` and J = D + S."""
        prob = self.plan.problem(y=y)
        if want_grad and grad is None:
            grad = torch.empty_like(y)
        if self.alpha > 0 and want_grad:  # one evaluation with the regulariser (sr_evaluate_reg)
            stats = self.plan.evaluate(prob, self.weights, self.cell_volume, grad, self.alpha, self.s_reg)
        else:
            stats = self.plan.evaluate(prob, self.weights, self.cell_volume, grad if want_grad else None)
        return stats, grad

    def value(self, y: torch.Tensor) -> float:
        stats, _ = self.evaluate(y, want_grad=False)
        return float(stats[0].item())

    def host_stats(self) -> dict:
        return self.plan.host_stats()

    def evaluate_host(self, y_host):
        """End-to-end evaluation from host memory: (J, dJ/dy) as (float, ndarray).

        ``y_host`` may be a numpy array (staged through an internal pinned buffer) or a pinned CPU
        ``torch.Tensor`` of the field's shape and dtype, which is copied to the device directly (the
        e2e contract: inputs already in pinned host memory).  The returned gradient is a view of an
        internal pinned buffer, overwritten by the next call."""
        shape = self.shape
        dt = self.frames.dtype
        if self._pinned_y is None:
            self._pinned_y = torch.empty(shape, dtype=dt, pin_memory=True)
            self._pinned_g = torch.empty(shape, dtype=dt, pin_memory=True)
            self._dev_y = torch.empty(shape, dtype=dt, device=self.frames.data.device)
            self._dev_g = torch.empty(shape, dtype=dt, device=self.frames.data.device)
        if isinstance(y_host, torch.Tensor) and y_host.device.type == "cpu" and y_host.is_pinned():
            if tuple(y_host.shape) != tuple(shape) or y_host.dtype != dt:
                raise ValueError(f"y must have shape {shape} and dtype {dt}")
            src = y_host.contiguous()
        else:
            y_host = np.asarray(y_host)
            if y_host.shape != shape:
                raise ValueError(f"y must have shape {shape}")
            self._pinned_y.numpy()[...] = y_host
            src = self._pinned_y
        self._dev_y.copy_(src, non_blocking=True)
        stats, g = self.evaluate(self._dev_y, self._dev_g)
        self._pinned_g.copy_(g, non_blocking=True)
        d = stats[0:1].to("cpu", non_blocking=False)
        value = float(d.item())
        if self.alpha > 0:
            value += float(self.s_reg.item())
        torch.cuda.current_stream().synchronize()
        return value, self._pinned_g.numpy()
