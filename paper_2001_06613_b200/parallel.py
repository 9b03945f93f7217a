"""Pixel-slab sharding across GPUs.

One process per GPU.  The image domain is cut into contiguous slabs of the slowest
memory axis (first axis fastest, grid.py:7-8, so a slab is one contiguous flat pixel
range).  Frames T_k are replicated; y and dD/dy are sharded, with ``halo_rows`` rows of
y on each side when the feature has a stencil (NGF: 2).  Per evaluation:

  pass 1 on the slab -> raw [G | s | vmax | -vmin | count]
  all-reduce (NCCL): SUM over G, s, count; MAX over vmax, -vmin   <- the only collective
  finalize (identical on every rank) -> C, D, gradient coefficients
  pass 2 on the slab -> this rank's dD/dy

Halo rows of y are refreshed with NCCL point-to-point before an evaluation that needs
them (exchange_halo).  The same code runs with world size 1 (no collective at all).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .engine import DeviceFrames, EvalPlan

__all__ = ["slab_ranges", "halo_range", "allreduce_raw", "exchange_halo", "ShardedFieldObjective"]


def slab_ranges(dims, world: int) -> list:
    """Flat pixel ranges [lo, hi) of ``world`` slabs along the slowest axis (rows split as
    evenly as possible, earlier ranks take the remainder)."""
    dims = tuple(int(d) for d in dims)
    rows = dims[-1]
    row = int(np.prod(dims[:-1]))
    if world < 1 or world > rows:
        raise ValueError(f"cannot split {rows} rows over {world} ranks")
    base, rem = divmod(rows, world)
    out, r0 = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((r0 * row, (r0 + n) * row))
        r0 += n
    return out


def halo_range(dims, lo: int, hi: int, halo_rows: int) -> tuple:
    row = int(np.prod(dims[:-1]))
    N = int(np.prod(dims))
    return max(0, lo - halo_rows * row), min(N, hi + halo_rows * row)


def allreduce_raw(raw: torch.Tensor, k: int, group=None) -> torch.Tensor:
    """In-place combination of the ranks' raw sums [G | s | vmax | -vmin | count] with ONE collective:
    an all-gather of the whole vector (K^2 + 3K + 1 doubles per rank), then, on every rank, the SUM over
    G, s and count and the MAX over the two extremum blocks in rank order.  The fixed order makes D and
    dD/dy bitwise identical on every rank and independent of the collective's internal reduction order."""
    if group is None:
        return raw
    world = dist.get_world_size(group)
    allr = torch.empty((world, raw.numel()), dtype=raw.dtype, device=raw.device)
    dist.all_gather(list(allr.unbind(0)), raw.contiguous(), group=group)
    kk = k * k + k
    acc = allr[0].clone()
    for r in range(1, world):  # fixed rank order
        acc[:kk] += allr[r, :kk]
        acc[kk:kk + 2 * k] = torch.maximum(acc[kk:kk + 2 * k], allr[r, kk:kk + 2 * k])
        acc[kk + 2 * k:] += allr[r, kk + 2 * k:]
    raw.copy_(acc)
    return raw


def exchange_halo(y_local: torch.Tensor, dims, lo: int, hi: int, halo_rows: int, group=None) -> None:
    """Refresh the halo rows of a [K, d, n_local] slab tensor from the neighbouring ranks."""
    if group is None or halo_rows == 0:
        return
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    row = int(np.prod(dims[:-1]))
    ylo, yhi = halo_range(dims, lo, hi, halo_rows)
    # NCCL moves device buffers directly; gloo's point-to-point needs host memory (CPU tests, gloo runs)
    stage = y_local.is_cuda and dist.get_backend(group) == "gloo"
    ops = []
    bufs = []
    # my first/last owned rows go to the neighbours' halos; their rows fill mine
    if rank > 0:
        n = min(halo_rows * row, hi - lo)
        send = y_local[..., lo - ylo:lo - ylo + n].contiguous()
        recv = torch.empty_like(y_local[..., :lo - ylo])
        if stage:
            send, recv = send.cpu(), recv.cpu()
        ops += [dist.P2POp(dist.isend, send, rank - 1, group), dist.P2POp(dist.irecv, recv, rank - 1, group)]
        bufs.append(("lo", recv))
    if rank < world - 1:
        n = min(halo_rows * row, hi - lo)
        send = y_local[..., hi - ylo - n:hi - ylo].contiguous()
        recv = torch.empty_like(y_local[..., hi - ylo:])
        if stage:
            send, recv = send.cpu(), recv.cpu()
        ops += [dist.P2POp(dist.isend, send, rank + 1, group), dist.P2POp(dist.irecv, recv, rank + 1, group)]
        bufs.append(("hi", recv))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    for side, buf in bufs:
        buf = buf.to(y_local.device)
        if side == "lo":
            y_local[..., :lo - ylo] = buf
        else:
            y_local[..., hi - ylo:] = buf


class ShardedFieldObjective:
    """D(y) and this rank's slab of dD/dy for a pixel-sharded displacement field."""

    def __init__(self, frames: DeviceFrames, frame_index, weights, cell_volume: float, *, feature: str = "ncc",
                 ngf_eps: float = 0.1, pix_range=None, halo_rows: int = 0, group=None):
        self.frames = frames
        self.grid = frames.grid
        N = self.grid.cell_count
        self.lo, self.hi = (0, N) if pix_range is None else (int(pix_range[0]), int(pix_range[1]))
        self.halo_rows = int(halo_rows) if feature == "ngf" else 0
        self.ylo, self.yhi = halo_range(self.grid.dims, self.lo, self.hi, max(self.halo_rows, 0))
        self.group = group
        self.feature = feature
        self.plan = EvalPlan(frames, frame_index, feature=feature, ngf_eps=ngf_eps, pix_range=(self.lo, self.hi))
        self.k = self.plan.k
        self.weights = np.asarray(weights, dtype=np.float64)
        self.cell_volume = float(cell_volume)
        self.whole = self.lo == 0 and self.hi == N and group is None

    def local_view(self, y_full: torch.Tensor) -> torch.Tensor:
        return y_full[..., self.ylo:self.yhi].contiguous()

    def launches_per_step(self) -> int:
        """Nominal engine launches per evaluate() (bench.py counts the real ones with CUPTI)."""
        if self.whole:  # sr_evaluate: pass 1 (2 kernels for fp32 NCC, K in 17..32), reduce + finalize, pass 2
            n = 3 + (1 if (self.feature == "ncc" and self.frames.data.dtype == torch.float32 and 17 <= self.k <= 32) else 0)
        else:  # pass 1, CTA reduce, finalize, pass 2
            n = 4
        if self.feature == "ngf":
            n += 1  # adjoint of the discrete gradient + chain rule
        return n

    def evaluate(self, y_local: torch.Tensor, grad_local: torch.Tensor):
        prob = self.plan.problem(y=y_local, y_off=self.ylo)
        if self.whole:
            return self.plan.evaluate(prob, self.weights, self.cell_volume, grad_local)
        exchange_halo(y_local, self.grid.dims, self.lo, self.hi, self.halo_rows, self.group)
        raw = self.plan.corr_partial(prob)
        allreduce_raw(raw, self.k, self.group)
        self.plan.finalize(prob, self.weights, self.cell_volume, n_total=self.grid.cell_count)
        self._grad(prob, grad_local)
        return self.plan.stats

    def _grad(self, prob, grad_local):
        """Pass 2 on the samples cached by this evaluation's pass 1 (y is unchanged in between)."""
        eng = self.frames.engine
        eng.set_sample_reuse(True)
        try:
            self.plan.grad(prob, grad_local, g_off=self.lo)
        finally:
            eng.set_sample_reuse(False)

    def kernel_times(self, y_local, grad_local, flush: torch.Tensor | None = None, reps: int = 20) -> dict:
        """Mean CUDA-event time (ms) of pass 1 (+ its CTA reduce), finalize (+ all-reduce when
        sharded) and pass 2, on the launching stream, L2 flushed before each evaluation."""
        prob = self.plan.problem(y=y_local, y_off=self.ylo)
        stream = torch.cuda.current_stream()
        acc = {"pass1": 0.0, "finalize": 0.0, "pass2": 0.0}
        for i in range(reps):
            if flush is not None:
                flush.fill_(float(i))
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(stream)
            raw = self.plan.corr_partial(prob)
            ev[1].record(stream)
            allreduce_raw(raw, self.k, self.group)
            self.plan.finalize(prob, self.weights, self.cell_volume, n_total=self.grid.cell_count)
            ev[2].record(stream)
            self._grad(prob, grad_local)
            ev[3].record(stream)
            torch.cuda.synchronize()
            acc["pass1"] += ev[0].elapsed_time(ev[1])
            acc["finalize"] += ev[1].elapsed_time(ev[2])
            acc["pass2"] += ev[2].elapsed_time(ev[3])
        return {k: v / reps for k, v in acc.items()}
