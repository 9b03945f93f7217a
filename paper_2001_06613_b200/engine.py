"""Device-side engine: one context per CUDA device, frame stacks resident in HBM,
and the evaluation plans that drive the C-ABI.

Layout in HBM:
  frames   [nframes][N]        dtype, first axis fastest (grid.py:7-8)
  shifts   [nframes]           dtype, frame means (raw-Gram centring shift)
  y, grad  [k][ndim][N]        dtype, absolute sample positions / dD/dy
  raw      [k*k + 2k + 1]      fp64 raw sums (all-reduced when pixels are sharded)
  stats    sr_stats_size(k)    fp64 C, sigma, D, gradient coefficients
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import (
    SR_AFFINE,
    SR_DISPLACEMENT,
    SR_F32,
    SR_F64,
    SR_NCC,
    SR_NGF,
    SrGrid,
    SrProblem,
    EngineUnavailable,
    check,
)

__all__ = [
    "Engine",
    "get_engine",
    "DeviceFrames",
    "GridSpec",
    "EvalPlan",
    "stats_view",
    "FEATURES",
    "DTYPES",
]

FEATURES = {"ncc": SR_NCC, "ngf": SR_NGF}
DTYPES = {torch.float32: SR_F32, torch.float64: SR_F64}


@dataclass(frozen=True)
class GridSpec:
    """Cell-centred grid (grid.py:61-99): dims, spacing, origin."""

    dims: tuple
    spacing: tuple
    origin: tuple

    @classmethod
    def of(cls, grid) -> "GridSpec":
        return cls(tuple(int(d) for d in grid.dims), tuple(float(s) for s in grid.spacing),
                   tuple(float(o) for o in grid.origin))

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def cell_count(self) -> int:
        return int(np.prod(self.dims))

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.spacing))

    def c_struct(self) -> SrGrid:
        g = SrGrid()
        g.ndim = self.ndim
        for a in range(3):
            g.dims[a] = self.dims[a] if a < self.ndim else 1
            g.spacing[a] = self.spacing[a] if a < self.ndim else 1.0
            g.origin[a] = self.origin[a] if a < self.ndim else 0.0
        return g


class Engine:
    """Owns one ``sr_ctx`` on one CUDA device."""

    def __init__(self, device: int | torch.device | None = None):
        if not torch.cuda.is_available():
            raise EngineUnavailable("no CUDA device: the seqreg B200 engine has no CPU path")
        self.lib = _lib.load_library()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", torch.device(device).index if not isinstance(device, int) else device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        ctx = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(self.lib.sr_create(self.device.index, ctypes.byref(ctx)))
        self.ctx = ctx
        self._frames: OrderedDict = OrderedDict()

    def __del__(self):
        try:
            if getattr(self, "ctx", None) is not None and self.lib is not None:
                self.lib.sr_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    def bind_stream(self, stream: torch.cuda.Stream | None = None) -> None:
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        check(self.lib.sr_set_stream(self.ctx, ctypes.c_void_p(s.cuda_stream)))

    def set_grid_ctas(self, ctas: int) -> None:
        check(self.lib.sr_set_grid_ctas(self.ctx, int(ctas)))

    def set_sample_reuse(self, enable: bool) -> None:
        """sr_grad may reuse the samples of the preceding sr_corr_partial (y unchanged in between)."""
        check(self.lib.sr_set_sample_reuse(self.ctx, 1 if enable else 0))

    # ------------------------------------------------------------------ frames
    def frames_for(self, seq, dtype: torch.dtype, cache_size: int = 8) -> "DeviceFrames":
        """Upload (once) and cache the frames of a reference ImageSequence."""
        key = (id(seq), dtype)
        hit = self._frames.get(key)
        if hit is not None and hit.owner is seq:
            self._frames.move_to_end(key)
            return hit
        values = np.stack([np.asarray(f.values, dtype=np.float64) for f in seq.frames])
        df = DeviceFrames.from_array(self, values, GridSpec.of(seq.grid), dtype)
        df.owner = seq
        self._frames[key] = df
        while len(self._frames) > cache_size:
            self._frames.popitem(last=False)
        return df


_ENGINES: dict = {}


def get_engine(device=None) -> Engine:
    if not torch.cuda.is_available():
        raise EngineUnavailable("no CUDA device: the seqreg B200 engine has no CPU path")
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    if idx is None:
        idx = torch.cuda.current_device()
    eng = _ENGINES.get(idx)
    if eng is None:
        eng = Engine(idx)
        _ENGINES[idx] = eng
    return eng


class DeviceFrames:
    """A frame stack resident on the device plus its per-frame shifts."""

    def __init__(self, engine: Engine, data: torch.Tensor, grid: GridSpec):
        if data.dim() != 2 or data.shape[1] != grid.cell_count:
            raise ValueError(f"frames must be [nframes, {grid.cell_count}]")
        if data.dtype not in DTYPES:
            raise ValueError("frames must be float32 or float64")
        self.engine = engine
        self.data = data.contiguous()
        self.grid = grid
        self.owner = None
        self.shifts = torch.empty(data.shape[0], dtype=data.dtype, device=data.device)
        engine.bind_stream()
        check(engine.lib.sr_frame_shifts(engine.ctx, DTYPES[data.dtype], ctypes.c_void_p(self.data.data_ptr()),
                                         int(data.shape[0]), int(data.shape[1]),
                                         ctypes.c_void_p(self.shifts.data_ptr())))

    @classmethod
    def from_array(cls, engine: Engine, values, grid: GridSpec, dtype: torch.dtype) -> "DeviceFrames":
        t = torch.as_tensor(np.ascontiguousarray(values)).to(device=engine.device, dtype=dtype)
        return cls(engine, t, grid)

    @property
    def nframes(self) -> int:
        return int(self.data.shape[0])

    @property
    def dtype(self) -> torch.dtype:
        return self.data.dtype


def stats_view(lib, stats: torch.Tensor, k: int) -> dict:
    """Split a host copy of the stats buffer into named arrays."""
    s = stats.detach().cpu().numpy() if isinstance(stats, torch.Tensor) else np.asarray(stats)
    off = {name: int(lib.sr_stats_offset(k, i)) for i, name in enumerate(
        ["C", "sigma", "mean", "vmax", "degen", "weights", "M", "beta", "shift"])}
    return {
        "D": float(s[0]),
        "corr": s[off["C"]:off["C"] + k * k].reshape(k, k).copy(),
        "sigma": s[off["sigma"]:off["sigma"] + k].copy(),
        "mean": s[off["mean"]:off["mean"] + k].copy(),
        "vmax": s[off["vmax"]:off["vmax"] + k].copy(),
        "degenerate": s[off["degen"]:off["degen"] + k] != 0,
        "weights": s[off["weights"]:off["weights"] + k].copy(),
        "M": s[off["M"]:off["M"] + k * k].reshape(k, k).copy(),
        "beta": s[off["beta"]:off["beta"] + k].copy(),
    }


class EvalPlan:
    """Everything one objective evaluation needs, kept alive for the C call.

    ``frame_index`` are 0-based frames in subset order.  For the affine
    parametrisation pass ``affine`` rows ([k, d*d+d] float64, host); for the
    displacement parametrisation pass ``y`` ([k, d, y_stride] on the device).
    """

    def __init__(self, frames: DeviceFrames, frame_index, *, feature: str = "ncc", ngf_eps: float = 0.1,
                 pix_range=None):
        self.frames = frames
        self.engine = frames.engine
        self.lib = frames.engine.lib
        self.grid = frames.grid
        self.k = len(frame_index)
        if self.k < 1:
            raise ValueError("subset must be nonempty")
        self.fidx = (ctypes.c_int32 * self.k)(*[int(i) for i in frame_index])
        if feature not in FEATURES:
            raise ValueError(f"feature must be one of {sorted(FEATURES)}")
        self.feature = feature
        self.ngf_eps = float(ngf_eps)
        N = self.grid.cell_count
        self.pix_range = (0, N) if pix_range is None else (int(pix_range[0]), int(pix_range[1]))
        dev = frames.data.device
        self.raw = torch.zeros(int(self.lib.sr_raw_size(self.k)), dtype=torch.float64, device=dev)
        self.stats = torch.zeros(int(self.lib.sr_stats_size(self.k)), dtype=torch.float64, device=dev)
        self._affine_buf = None
        self._keep = None

    def problem(self, *, affine=None, y: torch.Tensor | None = None, y_off: int = 0) -> SrProblem:
        p = SrProblem()
        p.grid = self.grid.c_struct()
        p.dtype = DTYPES[self.frames.dtype]
        p.feature = FEATURES[self.feature]
        p.ngf_eps = self.ngf_eps
        p.k = self.k
        p.frame_index = self.fidx
        p.frames_dev = self.frames.data.data_ptr()
        p.nframes = self.frames.nframes
        p.shifts_dev = self.frames.shifts.data_ptr()
        p.pix_lo, p.pix_hi = self.pix_range
        if affine is not None:
            a = np.ascontiguousarray(np.asarray(affine, dtype=np.float64).reshape(self.k, -1))
            d = self.grid.ndim
            if a.shape[1] != d * d + d:
                raise ValueError(f"expected {d * d + d} parameters per frame, got {a.shape[1]}")
            self._affine_buf = a
            p.param = SR_AFFINE
            p.affine = a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            p.y_dev = None
            p.y_stride = 1
        else:
            if y is None:
                raise ValueError("either affine parameters or a displacement field y is required")
            if y.dtype != self.frames.dtype or y.device != self.frames.data.device:
                raise ValueError("y must match the frames' dtype and device")
            if y.dim() != 3 or y.shape[0] != self.k or y.shape[1] != self.grid.ndim:
                raise ValueError(f"y must be [k={self.k}, d={self.grid.ndim}, n]")
            if not y.is_contiguous():
                raise ValueError("y must be contiguous")
            p.param = SR_DISPLACEMENT
            p.y_dev = y.data_ptr()
            p.y_off = int(y_off)
            p.y_stride = int(y.shape[2])
            p.affine = None
            self._keep = y
        return p

    # ---------------------------------------------------------------- the passes
    def sample(self, prob: SrProblem) -> torch.Tensor:
        """The warped values T_j(y_j(x)) of the problem's slab, [k, pix_hi - pix_lo] (sr_sample)."""
        out = torch.empty((self.k, int(prob.pix_hi - prob.pix_lo)), dtype=self.frames.dtype,
                          device=self.frames.data.device)
        self.engine.bind_stream()
        check(self.lib.sr_sample(self.engine.ctx, ctypes.byref(prob), ctypes.c_void_p(out.data_ptr())))
        return out

    def corr_partial(self, prob: SrProblem) -> torch.Tensor:
        self.engine.bind_stream()
        check(self.lib.sr_corr_partial(self.engine.ctx, ctypes.byref(prob), ctypes.c_void_p(self.raw.data_ptr())))
        return self.raw

    def finalize(self, prob: SrProblem, weights, cell_volume: float, n_total: int | None = None) -> torch.Tensor:
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        if w.size != self.k:
            raise ValueError("one weight per subset frame required")
        n_total = self.grid.cell_count if n_total is None else int(n_total)
        self.engine.bind_stream()
        check(self.lib.sr_corr_finalize(self.engine.ctx, ctypes.byref(prob), ctypes.c_void_p(self.raw.data_ptr()),
                                        w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), float(cell_volume),
                                        n_total, ctypes.c_void_p(self.stats.data_ptr())))
        return self.stats

    def grad(self, prob: SrProblem, out: torch.Tensor, g_off: int = 0) -> torch.Tensor:
        self.engine.bind_stream()
        stride = int(out.shape[-1]) if prob.param == SR_DISPLACEMENT else 0
        check(self.lib.sr_grad(self.engine.ctx, ctypes.byref(prob), ctypes.c_void_p(self.stats.data_ptr()),
                               ctypes.c_void_p(out.data_ptr()), int(g_off), stride))
        return out

    def evaluate(self, prob: SrProblem, weights, cell_volume: float, grad_out: torch.Tensor | None,
                 alpha: float = 0.0, s_out: torch.Tensor | None = None) -> torch.Tensor:
        """Whole evaluation on one device; returns the device stats (D = stats[0]).  alpha > 0 adds the
        curvature regulariser (sr_evaluate_reg): S in s_out[0], dS/dy added to grad_out."""
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        if w.size != self.k:
            raise ValueError("one weight per subset frame required")
        self.engine.bind_stream()
        wp = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        gp = ctypes.c_void_p(grad_out.data_ptr() if grad_out is not None else 0)
        if alpha > 0:
            check(self.lib.sr_evaluate_reg(self.engine.ctx, ctypes.byref(prob), wp, float(cell_volume), float(alpha),
                                           ctypes.c_void_p(self.raw.data_ptr()), ctypes.c_void_p(self.stats.data_ptr()),
                                           gp, ctypes.c_void_p(s_out.data_ptr())))
        else:
            check(self.lib.sr_evaluate(self.engine.ctx, ctypes.byref(prob), wp, float(cell_volume),
                                       ctypes.c_void_p(self.raw.data_ptr()), ctypes.c_void_p(self.stats.data_ptr()),
                                       gp))
        return self.stats

    def curvature(self, prob: SrProblem, alpha: float, cell_volume: float, grad: torch.Tensor,
                  s_out: torch.Tensor, g_off: int = 0) -> torch.Tensor:
        self.engine.bind_stream()
        check(self.lib.sr_curvature(self.engine.ctx, ctypes.byref(prob), float(alpha), float(cell_volume),
                                    ctypes.c_void_p(grad.data_ptr()), int(g_off), int(grad.shape[-1]),
                                    ctypes.c_void_p(s_out.data_ptr())))
        return s_out

    def host_stats(self) -> dict:
        return stats_view(self.lib, self.stats, self.k)
