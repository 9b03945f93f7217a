"""Minimal mirrors of the reference data types the hot path consumes.

The engine accepts the reference's own objects (``seqreg.Grid``, ``Image``,
``ImageSequence``, ``Affine``, ``AffineStack``) by duck typing; these mirrors
exist so the package is usable (and testable on a GPU box) without ``seqreg``
installed.  Semantics follow /root/reference/pkg/src/seqreg/grid.py:61-167 and
transform.py:35-178 (validation messages included).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Grid", "Image", "ImageSequence", "Affine", "AffineStack", "identity_affine", "identity_params"]


@dataclass(frozen=True)
class Grid:
    """Cell-centred rectilinear grid (grid.py:61-99)."""

    dims: tuple
    spacing: tuple
    origin: tuple

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        spacing = tuple(float(s) for s in self.spacing)
        origin = tuple(float(o) for o in self.origin)
        if not 1 <= len(dims) <= 3:
            raise ValueError(f"grid must be 1-, 2-, or 3-dimensional, got {len(dims)} axes")
        if len(spacing) != len(dims) or len(origin) != len(dims):
            raise ValueError("dims, spacing, and origin must have the same length")
        if any(d < 2 for d in dims):
            raise ValueError(f"all dims must be >= 2, got {dims}")
        if any(s <= 0 for s in spacing):
            raise ValueError(f"all spacings must be > 0, got {spacing}")
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "spacing", spacing)
        object.__setattr__(self, "origin", origin)

    @property
    def ndim(self) -> int:
        return len(self.dims)

    @property
    def cell_count(self) -> int:
        return int(np.prod(self.dims))

    @property
    def cell_volume(self) -> float:
        return float(np.prod(self.spacing))


class Image:
    """Grid plus one finite float64 value per cell, first axis fastest (grid.py:102-129)."""

    __slots__ = ("grid", "values")

    def __init__(self, grid: Grid, values):
        values = np.ascontiguousarray(values, dtype=np.float64).ravel()
        if values.size != grid.cell_count:
            raise ValueError(f"expected {grid.cell_count} values for dims {grid.dims}, got {values.size}")
        if not np.all(np.isfinite(values)):
            raise ValueError("image values must be finite")
        values.setflags(write=False)
        self.grid = grid
        self.values = values


class ImageSequence:
    """Frames on one grid with strictly increasing times (grid.py:132-167)."""

    __slots__ = ("grid", "frames", "times")

    def __init__(self, frames, times):
        frames = list(frames)
        times = tuple(float(t) for t in times)
        if len(frames) < 2:
            raise ValueError("a sequence needs at least 2 frames")
        if len(times) != len(frames):
            raise ValueError(f"{len(frames)} frames but {len(times)} times")
        grid = frames[0].grid
        if any(f.grid != grid for f in frames):
            raise ValueError("all frames must share one grid")
        if any(t1 <= t0 for t0, t1 in zip(times, times[1:])):
            raise ValueError("times must be strictly increasing")
        self.grid = grid
        self.frames = frames
        self.times = times

    @property
    def frame_count(self) -> int:
        return len(self.frames)


class Affine:
    """x -> A x + b; params are row-major vec(A) ++ b (transform.py:35-68)."""

    __slots__ = ("matrix", "translation")

    def __init__(self, matrix, translation):
        a = np.array(matrix, dtype=np.float64)
        b = np.array(translation, dtype=np.float64).ravel()
        if a.ndim != 2 or a.shape[0] != a.shape[1]:
            raise ValueError("matrix must be square")
        if b.size != a.shape[0]:
            raise ValueError("translation length must match matrix dimension")
        if not (np.all(np.isfinite(a)) and np.all(np.isfinite(b))):
            raise ValueError("affine entries must be finite")
        a.setflags(write=False)
        b.setflags(write=False)
        self.matrix = a
        self.translation = b

    @property
    def dim(self) -> int:
        return self.matrix.shape[0]

    @property
    def params(self) -> np.ndarray:
        return np.concatenate([self.matrix.ravel(), self.translation])

    @classmethod
    def from_params(cls, params, dim: int) -> "Affine":
        p = np.asarray(params, dtype=np.float64).ravel()
        if p.size != dim * dim + dim:
            raise ValueError(f"expected {dim * dim + dim} parameters, got {p.size}")
        return cls(p[: dim * dim].reshape(dim, dim), p[dim * dim:])


def identity_affine(d: int) -> Affine:
    if d not in (2, 3):
        raise ValueError(f"unsupported dimension {d}, expected 2 or 3")
    return Affine(np.eye(d), np.zeros(d))


def identity_params(d: int) -> np.ndarray:
    return np.concatenate([np.eye(d).ravel(), np.zeros(d)])


class AffineStack:
    """Per-frame transforms keyed by 1-based frame index (transform.py:117-178)."""

    __slots__ = ("items", "frame_count")

    def __init__(self, items: dict, frame_count: int):
        items = dict(items)
        if frame_count < 1:
            raise ValueError("frame_count must be >= 1")
        if not items:
            raise ValueError("stack must hold at least one transform")
        if len({t.dim for t in items.values()}) != 1:
            raise ValueError("all transforms must share one dimension")
        for k in items:
            if not 1 <= k <= frame_count:
                raise ValueError(f"frame index {k} outside 1..{frame_count}")
        self.items = items
        self.frame_count = frame_count

    @property
    def dim(self) -> int:
        return next(iter(self.items.values())).dim

    @property
    def indices(self) -> tuple:
        return tuple(sorted(self.items))

    def params_matrix(self) -> np.ndarray:
        return np.array([self.items[k].params for k in self.indices])

    def restrict(self, subset) -> "AffineStack":
        return AffineStack({k: self.items[k] for k in subset}, self.frame_count)

    @classmethod
    def identity(cls, frame_count: int, d: int, indices=None) -> "AffineStack":
        if indices is None:
            indices = range(1, frame_count + 1)
        return cls({k: identity_affine(d) for k in indices}, frame_count)

    @classmethod
    def from_params(cls, rows, indices, frame_count: int, dim: int) -> "AffineStack":
        rows = np.asarray(rows, dtype=np.float64)
        return cls({k: Affine.from_params(rows[i], dim) for i, k in enumerate(indices)}, frame_count)
