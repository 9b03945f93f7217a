"""Benchmark: voxel-frames/s of one D(y) + grad D(y) evaluation (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

A step is one objective evaluation (pass 1 warp+feature+Gram, fixed-order reduce,
finalize, pass 2 re-warp+coefficient contraction+chain rule) over the whole
workload with inputs resident in HBM.  Default workload: BASELINE.json configs[1]
("c2": 2-D, K=32, 512x512 float32, NCC, displacement-field iterate).  The inputs
(frames 33.5 MB + y 67 MB) fit in the 126 MB L2, so L2 is flushed (a 256 MiB write)
before every timed step, outside the step's CUDA-event window.

Multi-GPU (torchrun, one rank per GPU, NCCL): weak scaling — every rank owns a
512-row slab of a 512 x (512 N) domain (same per-GPU work), the K x K raw Gram sums
are all-reduced (the only collective), and each rank assembles its slab's gradient.

--impl reference: the CPU oracle port of the reference path (oracle/seqreg_oracle.py,
numpy, the reference's per-frame thread pool) on this host's cores, same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "voxel-frames/s for D(y)+∇D(y) eval at 1/2/4/8 GPU; % of HBM roofline"
# algorithmic bytes per voxel-frame, fp32 / fp64: pass 1 reads T (s) + y (d s);
# pass 2 reads T + y and writes dD/dy (d s)
def bytes_per_vf(d: int, s: int) -> dict:
    return {"pass1": (1 + d) * s, "pass2": (1 + 2 * d) * s, "eval": (2 + 3 * d) * s}


# compulsory bytes per voxel-frame of each engine kernel as designed: the split pass 1
# (k_sample_gram / k_sample_v) writes V (s) and grad T (d s) next to its y + T reads; the streaming pass 2
# reads them back and writes dD/dy; the fused kernels move exactly the SURVEY §8d pass figures
def kernel_bytes_per_vf(d: int, s: int) -> dict:
    return {"k_sample_v": 2 * (1 + d) * s, "k_gram_tc": s, "k_pass2_stream": (1 + 2 * d) * s,
            "k_sample_gram": 2 * (1 + d) * s, "k_sample_vp": 2 * (1 + d) * s, "k_pass2_tma": (1 + 2 * d) * s, "k_pass2_mma": (1 + 2 * d) * s, "k_gram_tma": s, "k_gram_mma": s,
            "k_pass2_bulk": (1 + 2 * d) * s,
            "k_pass2": (1 + 2 * d) * s, "k_pass1_tc": (1 + d) * s, "k_pass1_ws": (1 + d) * s, "k_pass1": (1 + d) * s,
            "k_reduce_finalize": 0,
            # split NGF path: u -> (n, rho); Gram of n; z from (n, rho); adjoint stencil of z with grad T
            "k_ngf_feat": (2 + d) * s, "k_gram_tcx": d * s, "k_ngf_z": (2 * d + 1) * s, "k_ngf_z_mma": (2 * d + 1) * s, "k_ngf_z_f16": (2 * d + 1) * s,
            "k_ngf_feat4": (2 + d) * s, "k_ngf_adj4": 3 * d * s,
            "k_ngf_adj_stream": 3 * d * s}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        j = json.loads(p.read_text())
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler running during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.002):
        self.samples = []
        self.period = period
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # pragma: no cover - depends on the box
            self.err = str(exc)
        self._stop = threading.Event()
        self.window = (0.0, 0.0)

    def _run(self):
        while not self._stop.is_set():
            try:
                t = time.perf_counter()
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                reasons = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((t, mhz, reasons))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.th.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": f"nvml unavailable: {self.err}"}
        t0, t1 = self.window
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        if len(inside) < 3:  # very short timed regions: take the samples nearest to the window
            mid = 0.5 * (t0 + t1)
            inside = sorted(self.samples, key=lambda s: abs(s[0] - mid))[:5]
        mhz = [s[1] for s in inside]
        bits = 0
        for s in inside:
            bits |= s[2]
        reasons = sorted({name for b, name in self.REASONS.items() if bits & b} - {"gpu_idle"})
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(inside)}


def build_workload(cfg_name: str, rank: int, world: int, device):
    """Synthetic inputs of the config, generated on the device. Weak scaling: the domain
    is world slabs tall (each rank owns one config-sized slab)."""
    import torch

    from paper_2001_06613_b200 import synth

    cfg = synth.CONFIGS[cfg_name]
    dims = list(cfg.dims)
    dims[-1] *= world
    dims = tuple(dims)
    frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device=device, dims=dims)
    y = synth.smooth_noise_iterate(dims, cfg.K, device=device) if cfg_name == "c2" else None
    if y is None:  # other configs evaluate at the true-motion-free identity plus smooth noise too
        y = synth.smooth_noise_iterate(dims, cfg.K, std_px=0.3, device=device)
    w = synth.config_weights(cfg)
    return cfg, dims, spacing, origin, frames.to(cfg.dtype), y.to(cfg.dtype).contiguous(), w


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2001_06613_b200 as srb
    from paper_2001_06613_b200.parallel import ShardedFieldObjective, slab_ranges

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg, dims, spacing, origin, frames, y_full, w = build_workload(args.config, rank, world, dev)
    d = len(dims)
    N = int(np.prod(dims))
    K = cfg.K
    eng = srb.get_engine(local)
    grid = srb.GridSpec(dims, spacing, origin)
    fd = srb.DeviceFrames(eng, frames, grid)
    h = grid.cell_volume
    lo, hi = slab_ranges(dims, world)[rank]
    obj = ShardedFieldObjective(fd, list(range(K)), w, h, feature=cfg.feature, ngf_eps=cfg.ngf_eps,
                                pix_range=(lo, hi), halo_rows=2 if cfg.feature == "ngf" else 0,
                                group=dist.group.WORLD if world > 1 else None)
    y = obj.local_view(y_full)
    del y_full
    grad = torch.empty((K, d, hi - lo), dtype=cfg.dtype, device=dev)
    vf_rank = (hi - lo) * K
    flush_w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flush_r = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    class _Flush:
        """Write 256 MiB (evicts the inputs) then read 256 MiB (writes the dirty lines back),
        so the timed step starts with a cold, clean L2."""

        def fill_(self, v):
            flush_w.fill_(v)
            flush_r.sum()

    flush = _Flush()
    stream = torch.cuda.current_stream()

    def step():
        obj.evaluate(y, grad)

    for _ in range(max(3, args.warmup)):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    launches_per_step, kdev = engine_kernel_times(step, flush, reps=max(5, min(args.steps, 20)))

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    with sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        t_wall1 = time.perf_counter()
        if world > 1:
            dist.barrier()
        sampler.window = (t_wall0, t_wall1)
    ms = [a.elapsed_time(b) for a, b in ev]
    ms_step = float(np.mean(ms))
    t = torch.tensor([ms_step], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    vf_total = N * K
    value = vf_total / (ms_step * 1e-3)

    # ---- roofline.  Phases by CUDA events on the launching stream (pass 1 = its kernels + CTA reduce,
    # finalize, pass 2 = one kernel); per kernel by CUPTI device time over the same flushed loop.  The
    # dominant kernel is the longest one; its bytes are its compulsory traffic per voxel-frame.
    rl = obj.kernel_times(y, grad, flush, reps=max(5, min(args.steps, 50)))
    s = 4 if cfg.dtype == torch.float32 else 8
    bpv = bytes_per_vf(d, s)
    kbv = kernel_bytes_per_vf(d, s)
    peak, peak_src = _peaks()
    kern = max(kdev, key=kdev.get)
    kern_ms = kdev[kern]
    achieved = kbv.get(kern, 0) * vf_rank / (kern_ms * 1e-3) / 1e9
    eval_achieved = bpv["eval"] * vf_rank / (ms_step * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / f"traffic_{args.config}.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(kern)

    # ---- e2e: the public host API (pinned H2D of y, evaluation, D2H of D and dD/dy)
    e2e = None
    if world == 1:
        # the step's input already in pinned host memory (the e2e contract); the timed region holds the
        # H2D of y, the evaluation and the D2H of D and dD/dy, every step
        y_host = y.cpu().pin_memory()
        fo = srb.FieldObjective(fd, list(range(K)), w, h, feature=cfg.feature, ngf_eps=cfg.ngf_eps)
        for _ in range(2):
            fo.evaluate_host(y_host)
        reps = max(3, min(args.steps, 20))
        t0 = time.perf_counter()
        for _ in range(reps):
            fo.evaluate_host(y_host)
        e2e_s = (time.perf_counter() - t0) / reps
        nbytes = int(y_host.numel() * y_host.element_size())
        e2e = {"value": vf_total / e2e_s, "unit": "voxel-frames/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes + 8, "ms_per_step": e2e_s * 1e3,
               "pcie_gbs": 2 * nbytes / e2e_s / 1e9}

    # ---- CPU baseline: the oracle port on a bounded sample (rank 0, N=1)
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(args.config, threads=1, budget_s=args.cpu_budget)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "voxel-frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if cfg.dtype == torch.float32 else "f64",
            "data": "synthetic (seeded Gaussian-blob sequence + sinusoidal motion, BASELINE.json generator)",
            "config": {"workload": f"{args.config}: {d}-D K={K} {'x'.join(map(str, cfg.dims))} "
                                   f"{'fp32' if s == 4 else 'fp64'} {cfg.feature.upper()} displacement-field D+grad eval",
                       "dims_global": list(dims), "frames": K, "feature": cfg.feature,
                       "parallelism": f"pixel slabs x{world} + NCCL all-reduce of the K x K raw Gram",
                       "l2": "flushed before every timed step (256 MiB write + 256 MiB read, outside the event window)"},
            "roofline": {"bound": "hbm", "kernel": kern, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "bytes_per_vf": kbv.get(kern, 0), "kernel_ms": kern_ms, "kernel_timing": "CUPTI device time",
                         "kernels_ms": kdev, "kernels_bytes_per_vf": {k: kbv.get(k, 0) for k in kdev},
                         "eval_achieved": eval_achieved, "eval_frac": eval_achieved / peak,
                         "eval_bytes_per_vf": bpv["eval"], "phases_ms_events": rl},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": sampler.summary(),
            "wall_s_timed_region": t_wall1 - t_wall0,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def engine_kernel_times(step, flush, reps: int = 10):
    """Kernels of the engine's .so (namespace sr::) per step and their mean CUPTI device time (ms),
    over ``reps`` steps with the L2 flush in between, outside the timed region."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(reps):
            flush.fill_(float(i))
            step()
        torch.cuda.synchronize()
    times, count = {}, 0
    for ev in prof.events():
        if ev.device_type.name == "CUDA" and "sr::" in ev.name:
            count += 1
            base = ev.name.replace("void ", "").replace("sr::", "").split("<")[0].split("(")[0].strip()
            times.setdefault(base, []).append(ev.device_time * 1e-3)
    return count // reps, {k: float(sum(v) / len(v)) for k, v in times.items()}


def cpu_baseline(config: str, threads: int, budget_s: float = 15.0, evals: int | None = None):
    """Time the CPU oracle (the reference algorithm restated in numpy) on the config's full
    workload; bounded by ``budget_s`` of evaluations (at least one)."""
    import torch

    from oracle import seqreg_oracle as orc
    from paper_2001_06613_b200 import synth

    cfg = synth.CONFIGS[config]
    frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device="cpu")
    y = synth.smooth_noise_iterate(cfg.dims, cfg.K, device="cpu")
    if cfg.dtype == torch.float32:
        fr = [f for f in frames.numpy().astype(np.float32).astype(np.float64)]
        yv = y.numpy().astype(np.float32).astype(np.float64)
    else:
        fr, yv = list(frames.numpy()), y.numpy()
    w = synth.config_weights(cfg)
    h = float(np.prod(spacing))
    vf = int(np.prod(cfg.dims)) * cfg.K
    times_s = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        orc.evaluate_field(fr, cfg.dims, spacing, origin, yv, w, h, cfg.feature, cfg.ngf_eps, threads=threads)
        times_s.append(time.perf_counter() - t0)
        if evals is not None and len(times_s) >= evals:
            break
        if evals is None and time.perf_counter() - t_start > budget_s:
            break
    best = float(np.median(times_s))
    return {"value": vf / best, "unit": "voxel-frames/s", "cores": threads, "kind": "port",
            "sample": f"full {config} evaluation ({vf} voxel-frames) x{len(times_s)}, numpy oracle "
                      f"(oracle/seqreg_oracle.py), median", "s_per_eval": best}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    import torch

    from oracle import seqreg_oracle as orc
    from paper_2001_06613_b200 import synth

    cfg = synth.CONFIGS[args.config]
    frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device="cpu")
    y = synth.smooth_noise_iterate(cfg.dims, cfg.K, device="cpu")
    fr = list(frames.numpy().astype(np.float32).astype(np.float64)) if cfg.dtype == torch.float32 else list(frames.numpy())
    yv = y.numpy().astype(np.float32).astype(np.float64) if cfg.dtype == torch.float32 else y.numpy()
    w = synth.config_weights(cfg)
    h = float(np.prod(spacing))
    vf = int(np.prod(cfg.dims)) * cfg.K
    run = lambda: orc.evaluate_field(fr, cfg.dims, spacing, origin, yv, w, h, cfg.feature, cfg.ngf_eps, threads=cores)
    for _ in range(max(1, min(args.warmup, 2))):
        run()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run()
        ts.append(time.perf_counter() - t0)
    s = float(np.mean(ts))
    value = vf / s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "voxel-frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": s * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64 arithmetic on f32-quantised inputs",
        "data": "synthetic (seeded Gaussian-blob sequence + sinusoidal motion, BASELINE.json generator)",
        "config": {"workload": f"{args.config}: {len(cfg.dims)}-D K={cfg.K} {'x'.join(map(str, cfg.dims))} "
                               f"{cfg.feature.upper()} displacement-field D+grad eval (CPU oracle port)"},
        "cpu_baseline": {"value": value, "unit": "voxel-frames/s", "cores": cores, "kind": "port",
                         "sample": f"full {args.config} evaluation per step, per-frame thread pool of {cores}"},
        "e2e": {"value": value, "unit": "voxel-frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
