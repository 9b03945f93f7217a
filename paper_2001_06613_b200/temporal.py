"""Temporal prolongation on the device (north_star kernel 4).

Generalises the reference's per-parameter-component predictors to fields of m
components per frame (m = d*d + d for affine stacks, m = d*N for displacement
fields), one independent problem per component:

  * ``ls_predict_fields``   temporal.py:194-239 — (M + beta L) zeta = M eta + beta L ref,
    tridiagonal, solved by the Thomas recurrences of thomas_solve (temporal.py:166-191).
    The matrix depends only on the mask and beta, so it is factorised once on the
    host and every component runs the substitution sweeps in one CUDA thread.
  * ``interp_linear_fields`` temporal.py:109-127 — theta-weighted blend of the
    bracketing source frames; sources are copied unchanged.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import check
from .engine import DTYPES, get_engine

__all__ = ["ls_predict_fields", "interp_linear_fields"]


def _as_2d(t: torch.Tensor, n: int) -> torch.Tensor:
    if t.shape[0] != n:
        raise ValueError(f"expected {n} frames, got {t.shape[0]}")
    if not t.is_contiguous():
        raise ValueError("fields must be contiguous")
    return t


def ls_predict_fields(eta: torch.Tensor, mask, ref: torch.Tensor, beta: float) -> torch.Tensor:
    """eta, ref: [n, ...] device tensors (rows of inactive frames of eta are ignored);
    mask: n booleans (the active subset).  Returns zeta like ref."""
    n = ref.shape[0]
    mask = np.asarray(mask, dtype=bool)
    if mask.size != n:
        raise ValueError(f"expected {n} mask entries, got {mask.size}")
    if beta <= 0:
        raise ValueError("beta must be > 0")
    eta = _as_2d(eta, n)
    ref = _as_2d(ref, n)
    if eta.shape != ref.shape or eta.dtype != ref.dtype:
        raise ValueError("eta and ref must have the same shape and dtype")
    m = ref[0].numel()
    eng = get_engine(ref.device)
    eng.bind_stream()
    zeta = torch.empty_like(ref)
    mk = np.ascontiguousarray(mask.astype(np.uint8))
    check(eng.lib.sr_ls_predict(eng.ctx, DTYPES[ref.dtype], int(n), int(m),
                                mk.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), float(beta),
                                ctypes.c_void_p(eta.data_ptr()), ctypes.c_void_p(ref.data_ptr()),
                                ctypes.c_void_p(zeta.data_ptr())))
    return zeta


def interp_linear_fields(src: torch.Tensor, sources, times) -> torch.Tensor:
    """src: [n, ...] with valid rows at the (0-based) ``sources`` frames; returns all n frames."""
    n = src.shape[0]
    src = _as_2d(src, n)
    times = np.asarray(times, dtype=np.float64)
    sources = sorted(int(s) for s in sources)
    srcset = set(sources)
    left = np.zeros(n, dtype=np.int32)
    right = np.full(n, -1, dtype=np.int32)
    theta = np.zeros(n, dtype=np.float64)
    for k in range(n):
        if k in srcset:
            left[k] = k
            continue
        lo = max(z for z in sources if z < k)
        hi = min(z for z in sources if z > k)
        left[k], right[k] = lo, hi
        theta[k] = (times[k] - times[lo]) / (times[hi] - times[lo])
    m = src[0].numel()
    eng = get_engine(src.device)
    eng.bind_stream()
    out = torch.empty_like(src)
    check(eng.lib.sr_interp_linear(eng.ctx, DTYPES[src.dtype], int(n), int(m),
                                   left.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                   right.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                   theta.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                   ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(out.data_ptr())))
    return out
