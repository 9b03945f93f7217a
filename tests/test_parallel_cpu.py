"""Multi-rank host logic of the pixel-slab sharding (paper_2001_06613_b200/parallel.py) on CPU:
world size 2 over gloo.  Each rank forms the raw sums of its slab with the oracle's sampling
(the GPU kernels are not involved here), all-reduces them with allreduce_raw, finalizes, and
must reproduce the whole-grid oracle D; the y halo exchange must reproduce the neighbour rows."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import seqreg_oracle as orc
from paper_2001_06613_b200.parallel import allreduce_raw, exchange_halo, halo_range, slab_ranges


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    rng = np.random.default_rng(0)
    from scipy.ndimage import gaussian_filter

    dims, K = (16, 12), 4
    spacing, origin = (0.5, 0.25), (-4.0, -1.5)
    frames = np.stack([gaussian_filter(rng.standard_normal(dims), 1.5).ravel(order="F") + 2.0 for _ in range(K)])
    x = orc.cell_centers(dims, spacing, origin).T
    y = x[None] + 0.3 * rng.standard_normal((K,) + x.shape) * np.asarray(spacing)[None, :, None]
    w = rng.uniform(0.5, 1.0, K)
    return dims, spacing, origin, frames, y, w


def _raw_partial(frames, dims, spacing, origin, y, lo, hi, shifts):
    """[G | s | vmax | -vmin | count] of the shifted warped values over pixels [lo, hi)."""
    K = frames.shape[0]
    V = np.empty((hi - lo, K))
    vals = np.empty((hi - lo, K))
    for k in range(K):
        v, _ = orc.interpolate(frames[k], dims, spacing, origin, y[k][:, lo:hi].T, False)
        vals[:, k] = v
        V[:, k] = v - shifts[k]
    return np.concatenate([(V.T @ V).ravel(), V.sum(0), vals.max(0), -vals.min(0), [hi - lo]])


def _finalize(raw, K, N, w, h):
    """Host restatement of finalize_block (engine.cuh) -> D."""
    G = raw[:K * K].reshape(K, K)
    s = raw[K * K:K * K + K]
    mu = s / N
    sig = np.sqrt(np.maximum(np.diag(G) - s * mu, 0.0))
    C = (G - np.outer(s, mu)) / np.outer(sig, sig)
    C = np.triu(C) + np.triu(C, 1).T
    m = np.outer(w, w) * C**2
    return max(0.0, h * ((w.sum() ** 2 - (w * w).sum()) - (m.sum() - np.trace(m))))


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, spacing, origin, frames, y, w = _problem()
        K, N = frames.shape[0], int(np.prod(dims))
        shifts = frames.mean(axis=1)
        lo, hi = slab_ranges(dims, world)[rank]
        raw = torch.as_tensor(_raw_partial(frames, dims, spacing, origin, y, lo, hi, shifts))
        allreduce_raw(raw, K, dist.group.WORLD)
        D = _finalize(raw.numpy(), K, N, w, float(np.prod(spacing)))
        # halo exchange of y rows (2 rows each side)
        ylo, yhi = halo_range(dims, lo, hi, 2)
        loc = torch.zeros((K, 2, yhi - ylo), dtype=torch.float64)
        loc[..., lo - ylo:hi - ylo] = torch.as_tensor(y[..., lo:hi])
        exchange_halo(loc, dims, lo, hi, 2, dist.group.WORLD)
        halo_ok = bool(torch.equal(loc, torch.as_tensor(y[..., ylo:yhi])))
        out[rank] = (D, int(raw[-1].item()), halo_ok)
    finally:
        dist.destroy_process_group()


def test_slab_ranges_cover_grid():
    for dims, world in [((16, 12), 2), ((512, 512), 8), ((128, 128, 128), 8), ((7, 5, 9), 4)]:
        r = slab_ranges(dims, world)
        assert r[0][0] == 0 and r[-1][1] == int(np.prod(dims))
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
        row = int(np.prod(dims[:-1]))
        assert all((hi - lo) % row == 0 for lo, hi in r)
    with pytest.raises(ValueError):
        slab_ranges((4, 3), 4)


def test_two_rank_allreduce_and_halo_gloo():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    dims, spacing, origin, frames, y, w = _problem()
    _, Dref, _ = orc.evaluate_field(list(frames), dims, spacing, origin, y, w, float(np.prod(spacing)))
    for rank in range(world):
        D, count, halo_ok = out[rank]
        assert count == int(np.prod(dims))
        assert D == pytest.approx(Dref, rel=1e-12)
        assert halo_ok
