"""STSQ1 sequences straight to the device.

Mirror of ``seqreg.grid.read_sequence`` / ``write_sequence`` (/root/reference/pkg/src/seqreg/grid.py:256-332):
same file format (ASCII header, blank line, little-endian float32 payload frame after frame), same
header checks, exception classes and messages.  The payload is read into pinned host memory and
copied to HBM once; the float64 widening the reference does with ``astype(np.float64)`` happens on
the device (exact).  ``write_sequence`` produces byte-identical files to the reference's writer.
"""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np
import torch

from .engine import DeviceFrames, GridSpec, get_engine

__all__ = [
    "SequenceFormatError",
    "MalformedHeaderError",
    "TruncatedPayloadError",
    "DimensionMismatchError",
    "read_sequence",
    "write_sequence",
]

_MAGIC = "STSQ1"  # grid.py:42
_HEADER_LIMIT = 1 << 20  # the header of any valid file is far shorter than this


class SequenceFormatError(ValueError):
    """grid.py:45-47."""


class MalformedHeaderError(SequenceFormatError):
    """grid.py:49-51."""


class TruncatedPayloadError(SequenceFormatError):
    """grid.py:53-55."""


class DimensionMismatchError(SequenceFormatError):
    """grid.py:57-59."""


def _check_grid(dims, spacing, origin):
    """The reference Grid's validation (grid.py:73-84), same ValueError messages."""
    if not 1 <= len(dims) <= 3:
        raise ValueError(f"grid must be 1-, 2-, or 3-dimensional, got {len(dims)} axes")
    if len(spacing) != len(dims) or len(origin) != len(dims):
        raise ValueError("dims, spacing, and origin must have the same length")
    if any(d < 2 for d in dims):
        raise ValueError(f"all dims must be >= 2, got {tuple(dims)}")
    if any(s <= 0 for s in spacing):
        raise ValueError(f"all spacings must be > 0, got {tuple(spacing)}")
    return GridSpec(tuple(int(d) for d in dims), tuple(float(s) for s in spacing), tuple(float(o) for o in origin))


def _header_field(lines, index, key):
    """grid.py:271-277."""
    if index >= len(lines):
        raise MalformedHeaderError(f"missing header line '{key}'")
    line = lines[index]
    if not line.startswith(key + ":"):
        raise MalformedHeaderError(f"expected header line '{key}: ...', got {line!r}")
    return line[len(key) + 1:].split()


def _parse_header(head: bytes):
    """grid.py:287-323, up to the payload size check."""
    try:
        lines = head.decode("ascii").split("\n")
    except UnicodeDecodeError as exc:
        raise MalformedHeaderError("header is not ASCII") from exc
    if not lines or lines[0] != _MAGIC:
        raise MalformedHeaderError(f"bad magic, expected {_MAGIC!r}")
    try:
        dims = [int(v) for v in _header_field(lines, 1, "dims")]
        spacing = [float(v) for v in _header_field(lines, 2, "spacing")]
        origin = [float(v) for v in _header_field(lines, 3, "origin")]
        (frames_str,) = _header_field(lines, 4, "frames")
        n = int(frames_str)
        times = [float(v) for v in _header_field(lines, 5, "times")]
    except (ValueError, TypeError) as exc:
        if isinstance(exc, SequenceFormatError):
            raise
        raise MalformedHeaderError(f"unparseable header: {exc}") from exc
    if not (len(dims) == len(spacing) == len(origin)):
        raise DimensionMismatchError(
            f"dims/spacing/origin lengths disagree: {len(dims)}/{len(spacing)}/{len(origin)}"
        )
    if len(times) != n:
        raise DimensionMismatchError(f"{n} frames declared but {len(times)} times given")
    try:
        grid = _check_grid(dims, spacing, origin)
    except ValueError as exc:
        raise MalformedHeaderError(f"invalid grid: {exc}") from exc
    return grid, n, times


def read_sequence(path, dtype: torch.dtype = torch.float64, engine=None):
    """Read an STSQ1 file into device memory.

    Returns ``(frames, times)``: a :class:`DeviceFrames` stack ``[n][N]`` of ``dtype`` on the engine's
    device and the frame times.  Errors are the reference's (grid.py:280-332).
    """
    path = Path(path)
    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head_chunk = fh.read(min(size, _HEADER_LIMIT))
        head, sep, _ = head_chunk.partition(b"\n\n")
        if not sep:
            raise MalformedHeaderError("no blank line terminating the header")
        grid, n, times = _parse_header(head)
        offset = len(head) + 2
        payload_len = size - offset
        expected = 4 * n * grid.cell_count
        if payload_len < expected:
            raise TruncatedPayloadError(f"payload has {payload_len} bytes, expected {expected}")
        if payload_len > expected:
            raise TruncatedPayloadError(f"payload has {payload_len - expected} trailing bytes")
        host = torch.empty(n * grid.cell_count, dtype=torch.float32, pin_memory=torch.cuda.is_available())
        fh.seek(offset)
        view = host.numpy().view(np.uint8)
        got = fh.readinto(memoryview(view))
        if got != expected:
            raise TruncatedPayloadError(f"payload has {got} bytes, expected {expected}")
    if not np.little_endian:  # the payload is "<f4" (grid.py:268)
        host = torch.from_numpy(host.numpy().byteswap())
    # the reference's Image / ImageSequence checks (grid.py:104-150), in its order, before any device work
    if not bool(torch.isfinite(host).all()):
        raise ValueError("image values must be finite")
    if n < 2:
        raise ValueError("a sequence needs at least 2 frames")
    if any(t1 <= t0 for t0, t1 in zip(times, times[1:])):
        raise ValueError("times must be strictly increasing")
    eng = engine if engine is not None else get_engine()
    dev = host.to(eng.device, non_blocking=True).reshape(n, grid.cell_count)
    data = dev if dtype == torch.float32 else dev.to(dtype)
    return DeviceFrames(eng, data.contiguous(), grid), [float(t) for t in times]


def write_sequence(frames: DeviceFrames, times, path) -> None:
    """Write a device stack in the STSQ1 format, byte-identical to grid.py:256-268."""
    g = frames.grid
    n = int(frames.data.shape[0])
    if len(times) != n:
        raise ValueError(f"{n} frames but {len(times)} times")
    header = "\n".join(
        [
            _MAGIC,
            "dims: " + " ".join(str(int(d)) for d in g.dims),
            "spacing: " + " ".join(repr(float(s)) for s in g.spacing),
            "origin: " + " ".join(repr(float(o)) for o in g.origin),
            f"frames: {n}",
            "times: " + " ".join(repr(float(t)) for t in times),
        ]
    )
    payload = frames.data.to(torch.float32).cpu().numpy().astype("<f4").tobytes()
    Path(path).write_bytes(header.encode("ascii") + b"\n\n" + payload)
