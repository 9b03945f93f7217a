"""Spatial hierarchy on the device.

* :func:`build_pyramid` mirrors ``seqreg.pyramid.build_pyramid`` (pyramid.py:68-91): the finest
  level is the input, each coarser level is restrict(smooth(frame)) for every frame, computed by
  ``sr_pyramid_step`` (bit-identical to the reference for fp64 stacks); same validation messages.
* :func:`prolong_field` carries a displacement field from a coarse level to the next finer one
  (``sr_prolong_field``; the reference has no displacement fields).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import check
from .engine import DTYPES, DeviceFrames, GridSpec

__all__ = ["coarse_grid", "pyramid_step", "build_pyramid", "prolong_field"]


def coarse_grid(grid: GridSpec) -> GridSpec:
    """pyramid.py:47-52: dims ceil(dims / 2), doubled spacing, same origin."""
    return GridSpec(tuple(-(-d // 2) for d in grid.dims), tuple(2.0 * s for s in grid.spacing), tuple(grid.origin))


def pyramid_step(frames: DeviceFrames) -> DeviceFrames:
    """restrict(smooth(f)) for every frame of the stack (pyramid.py:22-54)."""
    eng = frames.engine
    cg = coarse_grid(frames.grid)
    out = torch.empty((frames.data.shape[0], cg.cell_count), dtype=frames.data.dtype, device=frames.data.device)
    dims = (ctypes.c_int32 * 3)(*(list(frames.grid.dims) + [1] * (3 - frames.grid.ndim)))
    eng.bind_stream()
    check(eng.lib.sr_pyramid_step(eng.ctx, DTYPES[frames.data.dtype], frames.grid.ndim, dims,
                                  int(frames.data.shape[0]), ctypes.c_void_p(frames.data.data_ptr()),
                                  ctypes.c_void_p(out.data_ptr())))
    return DeviceFrames(eng, out, cg)


def build_pyramid(frames: DeviceFrames, level_count: int) -> list[DeviceFrames]:
    """pyramid.py:68-91: ``level_count`` levels ordered coarse to fine, the last one is ``frames``."""
    if level_count < 1:
        raise ValueError("level_count must be >= 1")
    dims = tuple(frames.grid.dims)
    for _ in range(level_count - 1):
        dims = tuple(-(-d // 2) for d in dims)
    if any(d < 4 for d in dims):
        raise ValueError(
            f"level_count={level_count} too large for dims {tuple(frames.grid.dims)}: "
            f"coarsest level would be {dims}"
        )
    levels = [frames]
    for _ in range(level_count - 1):
        levels.insert(0, pyramid_step(levels[0]))
    return levels


def prolong_field(y_coarse: torch.Tensor, coarse: GridSpec, fine: GridSpec) -> torch.Tensor:
    """[k, d, N_coarse] absolute positions on ``coarse`` -> [k, d, N_fine] on ``fine``:
    u = y - x interpolated multilinearly at the fine centres (clamped to the coarse hull)."""
    from .engine import get_engine

    if y_coarse.dim() != 3 or y_coarse.shape[1] != coarse.ndim or y_coarse.shape[2] != coarse.cell_count:
        raise ValueError(f"y must be [k, {coarse.ndim}, {coarse.cell_count}]")
    if y_coarse.dtype not in DTYPES or not y_coarse.is_cuda:
        raise ValueError("y must be a float32/float64 CUDA tensor")
    eng = get_engine(y_coarse.device)
    y = y_coarse.contiguous()
    out = torch.empty((y.shape[0], fine.ndim, fine.cell_count), dtype=y.dtype, device=y.device)
    gc, gf = coarse.c_struct(), fine.c_struct()
    eng.bind_stream()
    check(eng.lib.sr_prolong_field(eng.ctx, DTYPES[y.dtype], ctypes.byref(gc), ctypes.byref(gf), int(y.shape[0]),
                                   ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(out.data_ptr())))
    return out
