"""ShardedFieldObjective (paper_2001_06613_b200/parallel.py) with world size 2 on the B200: two processes
over gloo, each owning a pixel slab of the same problem on cuda:0 (the collective is the host-side gloo
all-gather, so no kernel waits on another rank's kernel).  Each rank runs pass 1 on its slab, combines the
raw sums with allreduce_raw, finalizes and runs pass 2 on its slab (NGF: halo rows refreshed by
exchange_halo); D must equal the whole-grid evaluation and the two gradient slabs must reassemble the
whole-grid gradient.  Tolerances: D 1e-12 (fp64) / 1e-6 (fp32) relative; gradients 1e-10 / 1e-5 of the
largest entry (the slab sums combine in another order than the single-device CTA tree)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = [("ncc", torch.float64, 7, (40, 36)), ("ncc", torch.float32, 20, (64, 48)),
         ("ngf", torch.float32, 6, (64, 48)), ("ngf", torch.float64, 5, (20, 18, 12))]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(dims, K, seed=3):
    from scipy.ndimage import gaussian_filter

    from oracle import seqreg_oracle as orc

    rng = np.random.default_rng(seed)
    spacing = tuple(1.0 / n for n in dims)
    origin = (0.0,) * len(dims)
    frames = np.stack([gaussian_filter(rng.standard_normal(dims), 1.5).ravel(order="F") + 2.0 for _ in range(K)])
    x = orc.cell_centers(dims, spacing, origin).T
    y = x[None] + 0.3 * rng.standard_normal((K,) + x.shape) * np.asarray(spacing)[None, :, None]
    w = rng.uniform(0.5, 1.0, K)
    return spacing, origin, frames, y, w


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2001_06613_b200 as srb
        from paper_2001_06613_b200.parallel import ShardedFieldObjective, slab_ranges

        feature, dtype, K, dims = case
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        spacing, origin, frames, y, w = _problem(dims, K)
        eng = srb.get_engine(0)
        grid = srb.GridSpec(dims, spacing, origin)
        fd = srb.DeviceFrames(eng, torch.as_tensor(frames, dtype=dtype).to(dev), grid)
        h = grid.cell_volume
        lo, hi = slab_ranges(dims, world)[rank]
        obj = ShardedFieldObjective(fd, list(range(K)), w, h, feature=feature, ngf_eps=0.3, pix_range=(lo, hi),
                                    halo_rows=2, group=dist.group.WORLD)
        y_full = torch.as_tensor(y, dtype=dtype).to(dev).contiguous()
        y_loc = obj.local_view(y_full)
        y_loc[..., :lo - obj.ylo] = 0  # halo rows start stale: exchange_halo must refresh them
        y_loc[..., hi - obj.ylo:] = 0
        g_loc = torch.empty((K, len(dims), hi - lo), dtype=dtype, device=dev)
        stats = obj.evaluate(y_loc, g_loc)
        torch.cuda.synchronize()
        out[rank] = (float(stats[0].item()), lo, hi, g_loc.double().cpu().numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{str(c[1])[-7:]}-K{c[2]}-{len(c[3])}d")
def test_two_rank_sharded_matches_whole_grid(case):
    import paper_2001_06613_b200 as srb

    feature, dtype, K, dims = case
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, case, out), nprocs=2, join=True, start_method="spawn")
    spacing, origin, frames, y, w = _problem(dims, K)
    dev = torch.device("cuda", 0)
    eng = srb.get_engine(0)
    fd = srb.DeviceFrames(eng, torch.as_tensor(frames, dtype=dtype).to(dev), srb.GridSpec(dims, spacing, origin))
    obj = srb.FieldObjective(fd, list(range(K)), w, feature=feature, ngf_eps=0.3)
    stats, g = obj.evaluate(torch.as_tensor(y, dtype=dtype).to(dev).contiguous())
    D = float(stats[0].item())
    g = g.double().cpu().numpy()
    tol_d, tol_g = (1e-12, 1e-10) if dtype == torch.float64 else (1e-6, 1e-5)
    gmax = np.abs(g).max()
    for rank in (0, 1):
        Dr, lo, hi, gr = out[rank]
        assert abs(Dr - D) <= tol_d * abs(D), (rank, Dr, D)
        assert np.abs(gr - g[..., lo:hi]).max() <= tol_g * gmax, rank
    assert out[0][2] == out[1][1] and out[0][1] == 0 and out[1][2] == int(np.prod(dims))
