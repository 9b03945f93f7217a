"""Drop-in replacement of the reference hot path (similarity.py:128-220) on the B200 engine.

Same names, argument meaning and error behaviour as
/root/reference/pkg/src/seqreg/similarity.py:

    correlation_state(seq, stack, subset, weights, cell_volume, threads=1)   (128-164)
    dissimilarity(state)                                                     (167-177)
    dissimilarity_gradient(state, seq, stack, subset, threads=1)             (180-220)

``threads`` is accepted and ignored (the device does the parallel work).  The
warp, feature, Gram, centring and gradient all run in the CUDA kernels of
``libseqreg_b200.so``; only K x K host arithmetic (``dissimilarity``) stays in
Python, exactly as in the reference.  ``install()`` rebinds the names that
``seqreg.temporal`` resolves at call time (temporal.py:35-41), so the
reference's multilevel drivers run unchanged on the GPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .engine import EvalPlan, get_engine

__all__ = [
    "CorrelationState",
    "configure",
    "correlation_state",
    "dissimilarity",
    "dissimilarity_gradient",
    "decompose",
    "min_consecutive_rho",
    "install",
    "uninstall",
]

_OPTIONS = {"dtype": torch.float64, "feature": "ncc", "ngf_eps": 0.1}


def configure(*, dtype=None, feature=None, ngf_eps=None) -> dict:
    """Set the arithmetic type (float64 = the reference's, float32) and feature (ncc/ngf)."""
    if dtype is not None:
        if dtype not in (torch.float32, torch.float64):
            raise ValueError("dtype must be torch.float32 or torch.float64")
        _OPTIONS["dtype"] = dtype
    if feature is not None:
        if feature not in ("ncc", "ngf"):
            raise ValueError("feature must be 'ncc' or 'ngf'")
        _OPTIONS["feature"] = feature
    if ngf_eps is not None:
        if not ngf_eps > 0:
            raise ValueError("ngf_eps must be > 0")
        _OPTIONS["ngf_eps"] = float(ngf_eps)
    return dict(_OPTIONS)


def _validate_subset(stack, subset) -> tuple:
    """similarity.py:90-99."""
    subset = tuple(int(k) for k in subset)
    if not subset:
        raise ValueError("subset must be nonempty")
    if any(k1 <= k0 for k0, k1 in zip(subset, subset[1:])):
        raise ValueError("subset indices must be strictly increasing")
    missing = [k for k in subset if k not in stack.items]
    if missing:
        raise ValueError(f"stack has no transform for frames {missing}")
    return subset


def _affine_rows(stack, subset) -> np.ndarray:
    rows = []
    for k in subset:
        t = stack.items[k]
        rows.append(np.concatenate([np.asarray(t.matrix, dtype=np.float64).ravel(),
                                    np.asarray(t.translation, dtype=np.float64).ravel()]))
    return np.ascontiguousarray(np.array(rows))


@dataclass
class CorrelationState:
    """Mirror of similarity.py:109-125.

    ``corr``, ``degenerate``, ``center_norms`` and ``weights`` are host arrays
    like the reference's.  The evaluation never materialises the N x K feature
    matrix (the gradient pass re-warps the frames on the device);
    ``features`` builds it on first access only: the device re-samples the warped
    values (sr_sample) and forms the reference's feature columns (similarity.py:73-87:
    centred, unit norm, zero for a degenerate frame; NGF: n / ||n|| over the d
    component images), returned as a host N x K (NGF: dN x K) array.
    """

    subset: tuple
    corr: np.ndarray
    weights: np.ndarray
    cell_volume: float
    degenerate: np.ndarray
    center_norms: np.ndarray
    means: np.ndarray = field(default=None, repr=False)
    _plan: EvalPlan = field(default=None, repr=False, compare=False)
    _prob: object = field(default=None, repr=False, compare=False)
    _prob_keep: object = field(default=None, repr=False, compare=False)  # the host affine rows _prob points at
    _features: np.ndarray = field(default=None, repr=False, compare=False)

    @property
    def features(self) -> np.ndarray:
        if self._features is None:
            if self._plan is None or self._prob is None:
                raise AttributeError("this state holds no device plan to materialise the features from")
            self._features = _materialise_features(self._plan, self._prob, self.degenerate)
        return self._features


def _materialise_features(plan: EvalPlan, prob, degenerate) -> np.ndarray:
    v = plan.sample(prob).to(torch.float64)  # [k, N]
    if plan.feature == "ngf":
        g = plan.grid
        u = v.reshape((v.shape[0],) + tuple(reversed(g.dims)))  # [k, n_{d-1}, ..., n_0] (first axis fastest)
        comps = []
        for ax in range(g.ndim):
            dim = u.dim() - 1 - ax
            n = u.shape[dim]
            up = torch.cat([u.narrow(dim, 1, n - 1), u.narrow(dim, n - 1, 1)], dim)
            um = torch.cat([u.narrow(dim, 0, 1), u.narrow(dim, 0, n - 1)], dim)
            scale = torch.full((n,), 0.5 / g.spacing[ax], dtype=torch.float64, device=u.device)
            scale[0] = scale[-1] = 1.0 / g.spacing[ax]  # one-sided at the domain edge
            shape = [1] * u.dim()
            shape[dim] = n
            comps.append((up - um) * scale.reshape(shape))
        p = torch.stack([c.reshape(v.shape[0], -1) for c in comps], dim=1)  # [k, d, N]
        nvec = p / torch.sqrt((p * p).sum(dim=1, keepdim=True) + plan.ngf_eps ** 2)
        f = nvec.reshape(v.shape[0], -1)
    else:
        f = v - v.mean(dim=1, keepdim=True)
    norms = torch.linalg.vector_norm(f, dim=1, keepdim=True)
    f = torch.where(norms > 0, f / torch.where(norms > 0, norms, 1.0), torch.zeros_like(f))
    deg = torch.as_tensor(np.asarray(degenerate, dtype=bool), device=f.device)
    f[deg] = 0.0
    return f.T.contiguous().cpu().numpy()


def correlation_state(seq, stack, subset, weights, cell_volume: float, threads: int = 1) -> CorrelationState:
    """Warp the subset frames, extract features, and correlate them (similarity.py:128-164)."""
    subset = _validate_subset(stack, subset)
    w = np.asarray(weights, dtype=np.float64)
    if w.size != len(subset):
        raise ValueError("one weight per subset frame required")
    if seq.grid.ndim != stack.dim:
        raise ValueError(f"points have dimension {seq.grid.ndim}, transform has {stack.dim}")
    eng = get_engine()
    frames = eng.frames_for(seq, _OPTIONS["dtype"])
    plan = EvalPlan(frames, [k - 1 for k in subset], feature=_OPTIONS["feature"], ngf_eps=_OPTIONS["ngf_eps"])
    prob = plan.problem(affine=_affine_rows(stack, subset))
    plan.corr_partial(prob)
    plan.finalize(prob, w, float(cell_volume))
    st = plan.host_stats()
    return CorrelationState(
        subset=subset,
        corr=st["corr"],
        weights=w,
        cell_volume=float(cell_volume),
        degenerate=st["degenerate"],
        center_norms=st["sigma"],
        means=st["mean"],
        _plan=plan,
        _prob=prob,
        _prob_keep=getattr(plan, "_affine_buf", None),
    )


def dissimilarity(state) -> float:
    """D = cell_volume * sum_{i != j} w_i w_j (1 - rho_ij^2), clamped at 0 (similarity.py:167-177)."""
    w = state.weights
    pair_mass = w.sum() ** 2 - (w * w).sum()
    m = np.outer(w, w) * state.corr**2
    coupling = m.sum() - np.trace(m)
    return max(0.0, state.cell_volume * (pair_mass - coupling))


def dissimilarity_gradient(state, seq, stack, subset, threads: int = 1) -> np.ndarray:
    """Analytic gradient w.r.t. the affine parameters, rows in subset order, vec(A) ++ b
    (similarity.py:180-220).  Degenerate frames give zero rows."""
    subset = _validate_subset(stack, subset)
    if subset != tuple(state.subset):
        raise ValueError("subset does not match the correlation state")
    plan = getattr(state, "_plan", None)
    if plan is None:
        raise ValueError("state was not produced by the B200 correlation_state")
    d = stack.dim
    prob = plan.problem(affine=_affine_rows(stack, subset))
    out = torch.empty(len(subset) * (d * d + d), dtype=torch.float64, device=plan.frames.data.device)
    plan.grad(prob, out)
    return out.cpu().numpy().reshape(len(subset), d * d + d)


def decompose(seq, stack, weights, cell_volume: float, inner_subset):
    """Within / within / cross split of D (similarity.py:223-253) on the engine's C."""
    all_frames = stack.indices
    inner = tuple(sorted(int(k) for k in inner_subset))
    if not inner or set(inner) - set(all_frames):
        raise ValueError("inner subset must be a nonempty subset of the stack's frames")
    if len(inner) == len(all_frames):
        raise ValueError("inner subset must be a proper subset")
    state = correlation_state(seq, stack, all_frames, weights, cell_volume)
    w = state.weights
    terms = np.outer(w, w) * (1.0 - state.corr**2)
    np.fill_diagonal(terms, 0.0)
    mask = np.isin(all_frames, inner)
    d_inner = cell_volume * terms[np.ix_(mask, mask)].sum()
    d_outer = cell_volume * terms[np.ix_(~mask, ~mask)].sum()
    d_mixed = cell_volume * (terms[np.ix_(mask, ~mask)].sum() + terms[np.ix_(~mask, mask)].sum())
    return float(d_inner), float(d_outer), float(d_mixed)


def min_consecutive_rho(seq, stack) -> float:
    """Minimum correlation between consecutive transformed frames (similarity.py:256-266)."""
    if seq.frame_count < 2:
        raise ValueError("need at least 2 frames")
    n = seq.frame_count
    state = correlation_state(seq, stack, tuple(range(1, n + 1)), np.ones(n), 1.0)
    return float(min(state.corr[i, i + 1] for i in range(n - 1)))


_SAVED: dict = {}


def install(module=None):
    """Rebind seqreg.temporal's hot-path names to the B200 engine.

    temporal.py imports correlation_state / dissimilarity / dissimilarity_gradient
    into its module globals (temporal.py:35-41) and resolves them at call time,
    so rebinding those three names routes every objective evaluation of
    ``_gir_solve`` and ``dissim_all_frames`` through the GPU.  ``seqreg.similarity``
    itself is left untouched (it stays the CPU oracle)."""
    if module is None:
        import seqreg.temporal as module  # noqa: PLC0415
    if id(module) not in _SAVED:
        _SAVED[id(module)] = (module, {n: getattr(module, n) for n in
                                       ("correlation_state", "dissimilarity", "dissimilarity_gradient")})
    module.correlation_state = correlation_state
    module.dissimilarity = dissimilarity
    module.dissimilarity_gradient = dissimilarity_gradient
    return module


def uninstall(module=None) -> None:
    if module is None:
        import seqreg.temporal as module  # noqa: PLC0415
    saved = _SAVED.pop(id(module), None)
    if saved is not None:
        for n, f in saved[1].items():
            setattr(saved[0], n, f)
