"""Spatio-temporal multilevel registration of displacement fields on the device (BASELINE C1 / C5).

The control flow is the reference's ``stml_run`` (/root/reference/pkg/src/seqreg/temporal.py:376-457)
with the affine stack replaced by the north_star parametrisation, per-cell sample positions
y_k(x) ([n, d, N], absolute positions, first axis fastest):

  * spatial levels, coarse to fine: ``build_pyramid`` (pyramid.py:69-91, ``sr_pyramid_step``); a level
    starts from the previous level's all-frames solution carried to the finer grid by
    ``prolong_field`` (the reference's affine stacks are grid independent);
  * temporal levels (``temporal_levels`` = build_temporal_levels, temporal.py:87-106), coarse to fine:
    solve on the active subset (``_solve`` = _gir_solve, temporal.py:304-341, with J = D + S: the
    north_star curvature regulariser S(y) in place of the affine drift penalty, no preconditioning
    scale), extend to all frames (``interp_linear_fields`` at the coarsest spatial level,
    ``ls_predict_fields`` after, temporal.py:413-420), score the extension over all frames
    (dissim_all_frames, temporal.py:297-301) and apply the reference's dissim stopping rule
    (check_stop, temporal.py:274-294; the finest spatial level always ends with the all-frames solve);
  * the solver is the device L-BFGS (``lbfgs_minimize``, optimizer.py:76-168) over the subset's
    fields in fp64, each objective call one fused D + grad D evaluation (+ S) on the device.

``FieldRunConfig`` mirrors RunConfig (config.py:15-46) where it applies.  BASELINE's "N Gauss-Newton
iterations per level" maps to ``OptimOptions(max_iters=N, grad_tol=f_tol=step_tol=1e-30)``.
The CPU checker with the same composition is ``oracle.seqreg_oracle.field_stml_run``.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .engine import DeviceFrames
from .field import FieldObjective
from .optimizer import ObjectiveEval, OptimOptions, lbfgs_minimize
from .spatial import build_pyramid, prolong_field
from .temporal import interp_linear_fields, ls_predict_fields

__all__ = ["FieldRunConfig", "FieldLevelRun", "temporal_levels", "default_time_interval", "quad_weights",
           "precondition_scale", "field_stml_run"]


def temporal_levels(n: int, coarsest_size: int) -> list:
    """build_temporal_levels (temporal.py:87-106) with 0-based frame indices, coarse to fine."""
    if n < 3:
        raise ValueError("need at least 3 frames")
    if coarsest_size < 3:
        raise ValueError("coarsest_size must be >= 3")
    levels = [tuple(range(n))]
    while len(levels[0]) > coarsest_size:
        finer = levels[0]
        strided = finer[::2]
        coarser = strided if strided[-1] == finer[-1] else strided + (finer[-1],)
        levels.insert(0, coarser)
        if len(strided) <= coarsest_size:
            break
    return levels


def default_time_interval(times) -> tuple:
    """similarity.py:42-47."""
    t = np.asarray(times, dtype=np.float64)
    half = 0.5 * (t[-1] - t[0]) / (len(t) - 1)
    return float(t[0] - half), float(t[-1] + half)


def quad_weights(times, a: float, b: float) -> np.ndarray:
    """similarity.py:50-70 (trapezoid weights on [a, b])."""
    t = np.asarray(times, dtype=np.float64)
    if t.size == 1:
        return np.array([b - a])
    w = np.empty(t.size)
    w[0] = (t[0] - a) + 0.5 * (t[1] - t[0])
    w[1:-1] = 0.5 * (t[2:] - t[:-2])
    w[-1] = 0.5 * (t[-1] - t[-2]) + (b - t[-1])
    return w


@dataclass
class FieldRunConfig:
    spatial_levels: int = 3
    temporal_coarsest_size: int = 3
    feature: str = "ngf"
    ngf_eps: float = 0.1
    alpha: float = 0.0            # curvature regulariser weight (S(y))
    weights: str = "quad"         # "quad": quad_weights over the full interval (temporal.py:313-314); "uniform": 1/n
    beta: float = 1e-5            # ls_predict smoothing (config.py:18)
    eps: float | None = 1e-3      # dissim stopping rule (config.py:20); None never skips a temporal level
    optim: OptimOptions = field(default_factory=OptimOptions)
    # The coarsest level starts from the cell centres shifted by start_offset cells along every axis.  The
    # reference starts its affine solves at the identity (temporal.py:365,416); for displacement fields the
    # identity puts every sample on an interpolation node, where T(y) is not differentiable (grid.py:204-208
    # picks the right-sided cell): the first line search then fails at every level (measured at C1: 0
    # iterations, line_search_failure) and the run is not reproducible to rounding.  0.3 cells stays off the
    # nodes after prolongation too (0.6, 1.2, 2.4 cells on the finer levels).  0 restores the identity.
    start_offset: float = 0.3
    # Preconditioned coordinates (the field analogue of _gir_solve's scale, temporal.py:320-325): the solver
    # sees x = y / c with c^2 = 1 / lambda_max(alpha h L^T L) = s^4 / (alpha h (4 d)^2) (s the smallest
    # spacing), so its unit first step (p = -g, optimizer.py:104) is stable for the stiffest curvature mode;
    # without it every C5 solve (alpha = 10) ends in line_search_failure at iteration 0.  c = 1 when alpha = 0.
    precondition: bool = True

    def __post_init__(self):
        if self.spatial_levels < 1:
            raise ValueError("spatial_levels must be >= 1")
        if self.temporal_coarsest_size < 3:
            raise ValueError("temporal_coarsest_size must be >= 3")
        if self.beta <= 0:
            raise ValueError("beta must be > 0")
        if self.eps is not None and self.eps <= 0:
            raise ValueError("eps must be > 0")
        if self.weights not in ("quad", "uniform"):
            raise ValueError("weights must be 'quad' or 'uniform'")
        if self.alpha < 0:
            raise ValueError("alpha must be >= 0")
        if not 0.0 <= self.start_offset < 1.0:
            raise ValueError("start_offset must be in [0, 1)")


@dataclass
class FieldLevelRun:
    """One solve (LevelRun, temporal.py:262-271)."""

    spatial_level: int
    temporal_level: int
    active: tuple
    iterations: int
    evaluations: int
    reason: str
    f_initial: float
    f_final: float
    dissim_all: float
    wall_ms: float
    y_init: object = None   # the solve's start and result ([k, d, N] device tensors) with keep_fields=True
    y_final: object = None


def _weights(cfg: FieldRunConfig, times, subset, interval, n: int) -> np.ndarray:
    if cfg.weights == "uniform":
        return np.full(len(subset), 1.0 / n)
    return quad_weights(np.asarray(times)[list(subset)], *interval)


def _identity(grid, n: int, dtype, device, offset: float = 0.0) -> torch.Tensor:
    axes = [grid.origin[a] + (np.arange(grid.dims[a]) + 0.5 + offset) * grid.spacing[a] for a in range(grid.ndim)]
    mesh = np.meshgrid(*axes, indexing="ij")
    x = np.stack([m.ravel(order="F") for m in mesh])
    return torch.as_tensor(x, dtype=dtype, device=device).unsqueeze(0).expand(n, -1, -1).contiguous()


def precondition_scale(grid, alpha: float) -> float:
    """c of FieldRunConfig.precondition: c^2 = s^4 / (alpha h (4 d)^2), 1 without the regulariser."""
    if alpha <= 0:
        return 1.0
    s = min(grid.spacing)
    return float(s * s / (4 * grid.ndim * np.sqrt(alpha * grid.cell_volume)))


def _solve(lvl: DeviceFrames, subset, init: torch.Tensor, w, cfg: FieldRunConfig):
    """_gir_solve (temporal.py:304-341) for displacement fields: J = D + S over the subset, in the
    preconditioned coordinates x = y / c."""
    obj = FieldObjective(lvl, list(subset), w, feature=cfg.feature, ngf_eps=cfg.ngf_eps, alpha=cfg.alpha)
    shape = obj.shape
    dt = lvl.dtype
    c = precondition_scale(lvl.grid, cfg.alpha) if cfg.precondition else 1.0
    y = torch.empty(shape, dtype=dt, device=lvl.data.device)
    g = torch.empty(shape, dtype=dt, device=lvl.data.device)

    def objective(x: torch.Tensor) -> ObjectiveEval:
        y.copy_(x.view(shape) * c if c != 1.0 else x.view(shape))
        stats, _ = obj.evaluate(y, g)
        value = stats[0] + obj.s_reg[0] if cfg.alpha > 0 else stats[0]
        grad = g.reshape(-1).to(torch.float64)
        return ObjectiveEval(float(value.item()), grad * c if c != 1.0 else grad)

    def evaluate_into(x: torch.Tensor, g_out: torch.Tensor) -> float:
        """The same objective without n-vector temporaries (the fields of C5's finest level are 1 GB in fp64):
        y = c x in one pass (the fp64 product rounded once into y's dtype, as above), the gradient scaled by c
        straight into the solver's fp64 buffer (an fp64 gradient exactly as above; an fp32 one is scaled in
        fp32 before the widening)."""
        if c != 1.0:
            torch.mul(x.view(shape), c, out=y)
        else:
            y.copy_(x.view(shape))
        stats, _ = obj.evaluate(y, g)
        value = stats[0] + obj.s_reg[0] if cfg.alpha > 0 else stats[0]
        if c != 1.0:
            torch.mul(g.reshape(-1), c, out=g_out)
        else:
            g_out.copy_(g.reshape(-1))
        return float(value.item())

    objective.evaluate_into = evaluate_into

    x0 = init.to(torch.float64).reshape(-1)
    x0 = (x0 / c if c != 1.0 else x0).contiguous()
    res = lbfgs_minimize(objective, x0, cfg.optim, engine=lvl.engine)
    xf = res.x_final.view(shape)
    return (xf * c if c != 1.0 else xf).to(dt), res


def _dissim_all(lvl: DeviceFrames, y_all: torch.Tensor, w_all, cfg: FieldRunConfig) -> float:
    """dissim_all_frames (temporal.py:297-301): D over all frames (no regulariser)."""
    obj = FieldObjective(lvl, list(range(y_all.shape[0])), w_all, feature=cfg.feature, ngf_eps=cfg.ngf_eps)
    return obj.value(y_all.contiguous())


def field_stml_run(frames: DeviceFrames, times, cfg: FieldRunConfig | None = None, *, trace=None,
                   keep_fields: bool = False):
    """Returns (y [n, d, N] on the finest grid, list of FieldLevelRun).  ``frames`` is the finest level;
    ``keep_fields`` records each solve's start and result fields in its FieldLevelRun."""
    cfg = cfg or FieldRunConfig()
    n = frames.nframes
    times = np.asarray(times, dtype=np.float64)
    if times.size != n:
        raise ValueError("one time per frame required")
    interval = default_time_interval(times)
    levels = temporal_levels(n, cfg.temporal_coarsest_size)
    t_final = len(levels) - 1
    pyramid = build_pyramid(frames, cfg.spatial_levels)
    dev, dt = frames.data.device, frames.dtype
    w_all = _weights(cfg, times, tuple(range(n)), interval, n)
    runs: list[FieldLevelRun] = []
    prev_full = None  # all-frames solution of the previous spatial level (its own grid)
    prev_grid = None
    for level, lvl in enumerate(pyramid):
        coarsest = level == 0
        finest = level == len(pyramid) - 1
        base = (_identity(lvl.grid, n, dt, dev, cfg.start_offset) if prev_full is None
                else prolong_field(prev_full, prev_grid, lvl.grid))
        history: list[FieldLevelRun] = []
        prediction = None
        current_full = None
        q = 0
        while q <= t_final:
            active = levels[q]
            idx = torch.as_tensor(active, device=dev)
            init = (base if q == 0 else prediction).index_select(0, idx)
            t0 = time.perf_counter()
            w = _weights(cfg, times, active, interval, n)
            y_q, res = _solve(lvl, active, init, w, cfg)
            if q == t_final:
                extension = y_q
            else:
                src = base.clone() if q == 0 else prediction.clone()
                src.index_copy_(0, idx, y_q)
                if coarsest:
                    extension = interp_linear_fields(src, active, times)
                else:
                    ref = base if q == 0 else prediction
                    mask = np.zeros(n, dtype=bool)
                    mask[list(active)] = True
                    extension = ls_predict_fields(src, mask, ref.contiguous(), cfg.beta)
            d_all = _dissim_all(lvl, extension, w_all, cfg)
            run = FieldLevelRun(level, q, tuple(active), res.iterations, res.objective_evaluations, res.converged_reason,
                                res.f_initial, res.f_final, d_all, 1e3 * (time.perf_counter() - t0),
                                init if keep_fields else None, y_q if keep_fields else None)
            runs.append(run)
            history.append(run)
            if trace is not None:
                trace(run)
            stop = False
            if cfg.eps is not None and 1 <= q < t_final:  # check_stop, dissim mode (temporal.py:286-288)
                stop = abs(history[-1].dissim_all - history[-2].dissim_all) <= cfg.eps * abs(history[0].dissim_all)
            current_full = extension
            if q < t_final:
                prediction = extension
            if stop:
                if finest:
                    q = t_final
                    continue
                break
            q += 1
        prev_full, prev_grid = current_full, lvl.grid
    return prev_full, runs
