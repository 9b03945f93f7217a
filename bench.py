"""Benchmark: voxel-frames/s of one D(y) + grad D(y) evaluation (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]

A step is one objective evaluation (pass 1: warp + feature + Gram; fixed-order reduce + finalize;
pass 2: re-warp + coefficient contraction + adjoint + chain rule) over the whole workload with the
inputs resident in HBM.  Default workload: configs[2] ("c3": 2-D, K = 100, 1024 x 1024 float32, NGF,
the largest single-GPU configuration, the one north_star names for 1/2/4/8 GPUs).  The same run also
measures c4 (3-D, K = 20, 128^3, NGF) and c2 (configs[1], K = 32, 512^2, NCC) and reports them under
"other_configs".  Inputs of every config are the seeded synthetic sequence (synth.make_sequence) and the
bench iterate (synth.bench_iterate: y = x + G_(4 px) * N(0, 0.5 px), the iterate every arm and the
full-size parity fixtures use).  c3 / c4 inputs (1.3 GB / 0.5 GB) exceed the 126 MB L2; every timed step
is still preceded by a 256 MiB write + 256 MiB read outside the event window (c2's inputs fit in L2).

--gpus N (N > 1): re-launches itself under torch.distributed.run (one rank per GPU, NCCL) unless already
inside a torchrun.  Strong scaling: the fixed config domain is cut into N slabs of the slowest axis
(pixels; frames replicated), the ranks' raw K x K Gram sums are combined by one all-gather (the only
collective), and each rank assembles its slab's gradient; value = all voxel-frames / max-over-ranks time.

--impl reference: the CPU restatement of the reference path (oracle/seqreg_oracle.py, numpy, the
reference's per-frame thread pool; the reference itself has neither NGF nor displacement fields) on all
host cores, on a bounded sample of the same config (a subset of the frames at full resolution).

--dry-run: no GPU work; checks the rank plumbing (gloo) and prints the line skeleton (CPU test).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "voxel-frames/s for D(y)+∇D(y) eval at 1/2/4/8 GPU; % of HBM roofline"


def bytes_per_vf(d: int, s: int) -> dict:
    """Algorithmic bytes per voxel-frame: pass 1 reads T (s) + y (d s); pass 2 reads T + y
    and writes dD/dy (d s).  2-D fp32: 12 + 20 = 32 B; 3-D fp32: 16 + 28 = 44 B."""
    return {"pass1": (1 + d) * s, "pass2": (1 + 2 * d) * s, "eval": (2 + 3 * d) * s}


# Each engine kernel's share of the algorithmic traffic: the kernel that gathers T at y for pass 1 is
# credited with pass 1's bytes, the one writing dD/dy with pass 2's, every other kernel with 0 (its
# traffic is intermediate data the fused two-pass design never materialises).  "own" = what the kernel
# itself must move as designed (the split kernels' intermediate reads / writes included).
def kernel_bytes_per_vf(d: int, s: int) -> dict:
    b = bytes_per_vf(d, s)
    alg = {"k_ngf_sfeat2": b["pass1"], "k_ngf_sfeat2f": b["pass1"], "k_sample_vp": b["pass1"], "k_pass2_tma": b["pass2"],
           "k_pass2_mma": b["pass2"], "k_ngf_adj4": b["pass2"], "k_pass1": b["pass1"], "k_pass2": b["pass2"]}
    own = {"k_ngf_sfeat2": (1 + d) * s + (3 * d + 1) * s,  # y, T in; n, 1/rho, grad T out
           "k_ngf_sfeat2f": (1 + d) * s + (3 * d + 1) * s,
           "k_sample_vp": 2 * (1 + d) * s, "k_pass2_tma": (1 + 2 * d) * s, "k_pass2_mma": (1 + 2 * d) * s,
           "k_gram_tma": s, "k_gram_h": d * s, "k_ngf_feat4": (3 + d) * s, "k_ngf_z_tc": (2 * d + 1) * s,
           "k_ngf_z_f16": (2 * d + 1) * s, "k_ngf_adj4": 3 * d * s, "k_pass1": b["pass1"], "k_pass2": b["pass2"],
           "k_reduce_finalize": 0}
    return {"algorithmic": alg, "own": own}


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


def build_workload(cfg_name: str, device):
    """Synthetic inputs of the config on the device: frames (synth.make_sequence, seed 0) and the bench
    iterate (synth.bench_iterate, seed 1), cast to the config dtype.  The whole domain on every rank
    (strong scaling: each rank then keeps its slab of y)."""
    from paper_2001_06613_b200 import synth

    cfg = synth.CONFIGS[cfg_name]
    frames, _, spacing, origin = synth.make_sequence(cfg, seed=0, device=device)
    y = synth.bench_iterate(cfg, device=device)
    w = synth.config_weights(cfg)
    return cfg, tuple(cfg.dims), spacing, origin, frames.to(cfg.dtype), y.to(cfg.dtype).contiguous(), w


class _Flush:
    """Write 256 MiB (evicts the inputs) then read 256 MiB (writes the dirty lines back), so the timed
    step starts with a cold, clean L2."""

    def __init__(self, dev):
        import torch

        self.w = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
        self.r = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def fill_(self, v):
        self.w.fill_(v)
        self.r.sum()


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
    return count // reps, {k: float(sum(v) / reps) for k, v in times.items()}


def measure_config(name: str, args, world: int, rank: int, dev, full: bool):
    """Time the config on this rank's slab; returns the per-config result dict (rank 0 fills it)."""
    import torch
    import torch.distributed as dist

    import paper_2001_06613_b200 as srb
    from paper_2001_06613_b200.parallel import ShardedFieldObjective, slab_ranges

    cfg, dims, spacing, origin, frames, y_full, w = build_workload(name, dev)
    d = len(dims)
    N = int(np.prod(dims))
    K = cfg.K
    eng = srb.get_engine(dev.index)
    grid = srb.GridSpec(dims, spacing, origin)
    fd = srb.DeviceFrames(eng, frames, grid)
    h = grid.cell_volume
    group = dist.group.WORLD if world > 1 else None
    lo, hi = slab_ranges(dims, world)[rank]
    obj = ShardedFieldObjective(fd, list(range(K)), w, h, feature=cfg.feature, ngf_eps=cfg.ngf_eps,
                                pix_range=(lo, hi), halo_rows=2 if cfg.feature == "ngf" else 0, group=group)
    y = obj.local_view(y_full)
    y_host = y_full.cpu().pin_memory() if (full and world == 1) else None
    del y_full
    grad = torch.empty((K, d, hi - lo), dtype=cfg.dtype, device=dev)
    vf_rank = (hi - lo) * K
    flush = _Flush(dev)
    stream = torch.cuda.current_stream()

    def step():
        obj.evaluate(y, grad)

    for _ in range(max(3, args.warmup)):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    launches_per_step, kdev = engine_kernel_times(step, flush, reps=max(3, min(args.steps, 10)))

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(dev.index)
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

    # ---- roofline of the dominant kernel on its ALGORITHMIC bytes (SURVEY §8d share), CUPTI device time
    # over the same flushed loop; the whole evaluation on 32 B (2-D) / 44 B (3-D) per voxel-frame
    s = 4 if cfg.dtype == torch.float32 else 8
    bpv = bytes_per_vf(d, s)
    kb = kernel_bytes_per_vf(d, s)
    peak, peak_src = _peaks()
    kern = max(kdev, key=kdev.get)
    kern_ms = kdev[kern]
    achieved = kb["algorithmic"].get(kern, 0) * vf_rank / (kern_ms * 1e-3) / 1e9
    eval_achieved = bpv["eval"] * vf_total / (ms_step * 1e-3) / 1e9 / world
    traffic = None
    prof = ROOT / "profiles" / f"traffic_{name}.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(kern)
    res = {
        "config": name, "value": value, "ms_per_step": ms_step, "n_gpus": world,
        "workload": f"{name}: {d}-D K={K} {'x'.join(map(str, dims))} {'fp32' if s == 4 else 'fp64'} "
                    f"{cfg.feature.upper()} displacement-field D+grad eval",
        "launches_per_step": launches_per_step,
        "roofline": {"bound": "hbm", "kernel": kern, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_vf": kb["algorithmic"].get(kern, 0), "kernel_ms": kern_ms,
                     "kernel_timing": "CUPTI device time, L2 flushed before each step",
                     "kernels_ms": kdev, "kernels_share": {k: v / sum(kdev.values()) for k, v in kdev.items()},
                     "kernels_own_bytes_per_vf": {k: kb["own"].get(k) for k in kdev},
                     "eval_achieved": eval_achieved, "eval_frac": eval_achieved / peak,
                     "eval_bytes_per_vf": bpv["eval"],
                     "eval_note": "algorithmic bytes of the whole evaluation (SURVEY §8d) / event-timed step, per GPU"},
        "clocks": sampler.summary(), "wall_s_timed_region": t_wall1 - t_wall0,
    }
    if full and world == 1:
        # ---- e2e: the public host API (FieldObjective.evaluate_host: pinned H2D of y, evaluation, D2H of
        # D and dD/dy), every step
        fo = srb.FieldObjective(fd, list(range(K)), w, h, feature=cfg.feature, ngf_eps=cfg.ngf_eps)
        for _ in range(2):
            fo.evaluate_host(y_host)
        reps = max(3, min(args.steps, 10))
        t0 = time.perf_counter()
        for _ in range(reps):
            fo.evaluate_host(y_host)
        e2e_s = (time.perf_counter() - t0) / reps
        nbytes = int(y_host.numel() * y_host.element_size())
        res["e2e"] = {"value": vf_total / e2e_s, "unit": "voxel-frames/s", "h2d_bytes_per_step": nbytes,
                      "d2h_bytes_per_step": nbytes + 8, "ms_per_step": e2e_s * 1e3,
                      "pcie_gbs": 2 * nbytes / e2e_s / 1e9,
                      "api": "FieldObjective.evaluate_host (pinned host y in, host D and dD/dy out)"}
    del obj, fd, frames, y, grad, flush
    torch.cuda.empty_cache()
    return res


def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    main_res = measure_config(args.config, args, world, rank, dev, full=True)
    others = {}
    for extra in ([] if args.only else [c for c in ("c4", "c2") if c != args.config]):
        r = measure_config(extra, args, world, rank, dev, full=False)
        others[extra] = {k: r[k] for k in ("workload", "value", "ms_per_step", "launches_per_step")}
        others[extra]["roofline"] = {k: r["roofline"][k] for k in
                                     ("kernel", "frac", "eval_frac", "kernels_ms", "eval_achieved")}
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu:
        cpu = cpu_baseline(args.config, threads=1, budget_s=args.cpu_budget)
    if rank == 0:
        from paper_2001_06613_b200 import synth

        cfg = synth.CONFIGS[args.config]
        line = {
            "metric": METRIC, "value": main_res["value"], "unit": "voxel-frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": main_res["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if cfg.dtype.itemsize == 4 else "f64",
            "data": "synthetic (seeded Gaussian-blob sequence + sinusoidal motion, BASELINE.json generator; "
                    "iterate synth.bench_iterate)",
            "config": {"workload": main_res["workload"], "dims": list(cfg.dims), "frames": cfg.K,
                       "feature": cfg.feature,
                       "parallelism": f"pixel slabs x{world}, frames replicated, one all-gather of the K x K raw "
                                      f"Gram sums per evaluation" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (c3/c4); 256 MiB write + read flush before every timed step "
                             "anyway, outside the event window"},
            "roofline": main_res["roofline"],
            "cpu_baseline": cpu,
            "e2e": main_res.get("e2e"),
            "gpu_launches": main_res["launches_per_step"] * args.steps,
            "clocks": main_res["clocks"],
            "wall_s_timed_region": main_res["wall_s_timed_region"],
            "other_configs": others,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _oracle_inputs(config: str, k_sample: int | None):
    """The config's inputs on the CPU (frames fp32-quantised, the bench iterate), optionally only the
    first ``k_sample`` frames (a bounded sample of the same workload: full resolution, fewer frames)."""
    import torch

    from paper_2001_06613_b200 import synth

    cfg = synth.CONFIGS[config]
    K = cfg.K if k_sample is None else min(cfg.K, k_sample)
    frames, _, spacing, origin = synth.make_sequence(cfg, seed=0, device="cpu", K=cfg.K)
    y = synth.smooth_noise_iterate(cfg.dims, cfg.K, sigma_px=4.0, std_px=0.5, seed=1)  # = synth.bench_iterate
    q = cfg.dtype == torch.float32
    fr = frames.numpy()[:K]
    yv = y.numpy()[:K]
    if q:
        fr = fr.astype(np.float32).astype(np.float64)
        yv = yv.astype(np.float32).astype(np.float64)
    w = synth.config_weights(cfg)[:K]
    return cfg, list(fr), yv, w, spacing, origin, K


def cpu_baseline(config: str, threads: int, budget_s: float = 15.0):
    """The CPU oracle (the reference algorithm restated in numpy) on one core, on a bounded sample of the
    config: the first K_s frames at full resolution, K_s sized for ~budget_s of work."""
    from oracle import seqreg_oracle as orc

    cfg, fr, yv, w, spacing, origin, _ = _oracle_inputs(config, None)
    h = float(np.prod(spacing))
    N = int(np.prod(cfg.dims))

    def run(k):
        t0 = time.perf_counter()
        orc.evaluate_field(fr[:k], cfg.dims, spacing, origin, yv[:k], w[:k], h, cfg.feature, cfg.ngf_eps,
                           threads=threads)
        return time.perf_counter() - t0

    k0 = min(cfg.K, 2)
    t1 = run(k0)
    ks = int(max(2, min(cfg.K, k0 * budget_s / max(t1, 1e-3))))
    ts = [run(ks)]
    s = float(np.median(ts))
    return {"value": N * ks / s, "unit": "voxel-frames/s", "cores": threads, "kind": "port",
            "sample": f"{config} with its first {ks} of {cfg.K} frames at full resolution ({N * ks} voxel-frames), "
                      f"numpy oracle (oracle/seqreg_oracle.py), one evaluation", "s_per_eval": s}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    from oracle import seqreg_oracle as orc

    cfg, fr, yv, w, spacing, origin, _ = _oracle_inputs(args.config, None)
    h = float(np.prod(spacing))
    N = int(np.prod(cfg.dims))

    def run(k):
        t0 = time.perf_counter()
        orc.evaluate_field(fr[:k], cfg.dims, spacing, origin, yv[:k], w[:k], h, cfg.feature, cfg.ngf_eps,
                           threads=cores)
        return time.perf_counter() - t0

    # each step a bounded sample (the first K_s frames at full resolution) sized so the whole
    # --warmup + --steps run takes about args.ref_budget seconds
    k0 = min(cfg.K, max(2, cores))
    t1 = run(k0)
    per_step = args.ref_budget / max(1, args.steps + min(args.warmup, 2))
    ks = int(max(2, min(cfg.K, k0 * per_step / max(t1, 1e-3))))
    for _ in range(max(0, min(args.warmup, 2) - 1)):
        run(ks)
    ts = [run(ks) for _ in range(args.steps)]
    s = float(np.mean(ts))
    value = N * ks / s
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "voxel-frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 arithmetic on f32-quantised inputs",
        "data": "synthetic (seeded Gaussian-blob sequence + sinusoidal motion, BASELINE.json generator)",
        "config": {"workload": f"{args.config}: {len(cfg.dims)}-D K={cfg.K} {'x'.join(map(str, cfg.dims))} "
                               f"{cfg.feature.upper()} displacement-field D+grad eval (CPU oracle port)"},
        "cpu_baseline": {"value": value, "unit": "voxel-frames/s", "cores": cores, "kind": "port",
                         "sample": f"per step: the first {ks} of {cfg.K} frames at full resolution "
                                   f"({N * ks} voxel-frames), per-frame thread pool of {cores}"},
        "e2e": {"value": value, "unit": "voxel-frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


PIPELINES = {
    # BASELINE configs[0] and configs[4]: the full spatio-temporal multilevel run (multilevel.field_stml_run)
    "c1": dict(spatial_levels=3, temporal_coarsest_size=4, iters=20),
    "c5": dict(spatial_levels=4, temporal_coarsest_size=9, iters=10),
}


def run_pipeline(args):
    """--pipeline: the end-to-end multilevel registration of C1 / C5 on one GPU.  A step is one whole run
    (every spatial x temporal level, fixed L-BFGS iterations) from the frames in pinned host memory to the
    final fields back in host memory; ``value`` counts the voxel-frames of every objective evaluation of
    the run per second of the run.  The final all-frames D is checked against the CPU oracle evaluated at
    the GPU's final fields (fp64 arithmetic on the same inputs)."""
    import torch

    import paper_2001_06613_b200 as srb
    from paper_2001_06613_b200 import multilevel as ml
    from paper_2001_06613_b200 import synth
    from paper_2001_06613_b200.optimizer import OptimOptions

    name = args.config
    if name not in PIPELINES:
        raise SystemExit(f"--pipeline runs {sorted(PIPELINES)}")
    pc = PIPELINES[name]
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device=dev)
    host = frames.to(cfg.dtype).cpu().pin_memory()
    del frames
    fcfg = ml.FieldRunConfig(spatial_levels=pc["spatial_levels"], temporal_coarsest_size=pc["temporal_coarsest_size"],
                             feature=cfg.feature, ngf_eps=cfg.ngf_eps, alpha=cfg.alpha, weights="uniform", eps=None,
                             optim=OptimOptions(max_iters=pc["iters"], grad_tol=1e-30, f_tol=1e-30, step_tol=1e-30))
    eng = srb.get_engine(0)
    grid = srb.GridSpec(cfg.dims, spacing, origin)

    out_host = []  # pinned result buffer, allocated by the first run (a pageable y.cpu() of C5's 537 MB of
                   # fields cost 0.24 s of a 0.5 s run)

    def one_run():
        fd = srb.DeviceFrames(eng, host.to(dev, non_blocking=True), grid)
        y, runs = ml.field_stml_run(fd, times, fcfg)
        if not out_host:
            out_host.append(torch.empty(y.shape, dtype=y.dtype, pin_memory=True))
        out_host[0].copy_(y, non_blocking=True)
        torch.cuda.synchronize()
        return out_host[0], runs

    for _ in range(max(1, args.warmup)):
        one_run()
    torch.cuda.synchronize()
    walls, last = [], None
    sampler = ClockSampler(0)
    with sampler:
        t_all = time.perf_counter()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            last = one_run()
            walls.append(time.perf_counter() - t0)
        sampler.window = (t_all, time.perf_counter())
    y_host, runs = last
    # voxel-frames evaluated per run: every objective evaluation of every solve + the all-frames scores
    levels_n = []
    dims = tuple(cfg.dims)
    for _ in range(pc["spatial_levels"]):
        levels_n.insert(0, int(np.prod(dims)))
        dims = tuple(-(-d // 2) for d in dims)
    vf = sum(levels_n[r.spatial_level] * (len(r.active) * r.evaluations + cfg.K) for r in runs)
    wall = float(np.median(walls))
    # final D against the oracle at the same fields (finest level, all frames, fp64 arithmetic)
    from oracle import seqreg_oracle as orc

    t0 = time.perf_counter()
    fr = host.double().numpy()
    _st, d_ref, _g = orc.evaluate_field(list(fr), cfg.dims, spacing, origin, y_host.double().numpy(),
                                        np.full(cfg.K, 1.0 / cfg.K), float(np.prod(spacing)), cfg.feature,
                                        cfg.ngf_eps, threads=os.cpu_count() or 8)
    oracle_s = time.perf_counter() - t0
    d_gpu = runs[-1].dissim_all
    nbytes_in = int(host.numel() * host.element_size())
    line = {
        "metric": METRIC, "value": vf / wall, "unit": "voxel-frames/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if cfg.dtype.itemsize == 4 else "f64",
        "data": "synthetic (seeded Gaussian-blob sequence + sinusoidal motion, BASELINE.json generator)",
        "config": {"workload": f"{name}: end-to-end multilevel run, {pc['spatial_levels']} spatial x "
                               f"{len(ml.temporal_levels(cfg.K, pc['temporal_coarsest_size']))} temporal levels, "
                               f"{pc['iters']} L-BFGS iterations per level, K={cfg.K} "
                               f"{'x'.join(map(str, cfg.dims))} {cfg.feature.upper()} alpha={cfg.alpha}",
                   "step": "one whole run: H2D of the frames, pyramid, every solve, D2H of the final fields"},
        "pipeline": {"runs": [{"level": [r.spatial_level, r.temporal_level], "frames": len(r.active),
                               "iterations": r.iterations, "evaluations": r.evaluations, "reason": r.reason,
                               "f_final": r.f_final, "dissim_all": r.dissim_all, "ms": r.wall_ms} for r in runs],
                     "voxel_frames_evaluated": vf, "wall_s": walls,
                     "final_D": d_gpu, "final_D_oracle": d_ref, "final_D_rel_err": abs(d_gpu - d_ref) / abs(d_ref),
                     "oracle_eval_s": oracle_s},
        "e2e": {"value": vf / wall, "unit": "voxel-frames/s", "h2d_bytes_per_step": nbytes_in,
                "d2h_bytes_per_step": int(y_host.numel() * y_host.element_size()), "ms_per_step": wall * 1e3},
        "clocks": sampler.summary(),
    }
    print(json.dumps(line), flush=True)


def run_dry(args):
    """CPU check of the multi-rank plumbing: every rank joins a gloo group, takes its slab of the config
    and checks the all-gather; rank 0 prints the line skeleton with n_gpus."""
    import torch
    import torch.distributed as dist

    from paper_2001_06613_b200 import synth
    from paper_2001_06613_b200.parallel import allreduce_raw, slab_ranges

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    cfg = synth.CONFIGS[args.config]
    lo, hi = slab_ranges(cfg.dims, world)[rank]
    K = cfg.K
    raw = torch.zeros(K * K + 3 * K + 1, dtype=torch.float64)
    raw[-1] = hi - lo
    allreduce_raw(raw, K, dist.group.WORLD if world > 1 else None)
    assert int(raw[-1].item()) == int(np.prod(cfg.dims)), "slabs do not cover the domain"
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "voxel-frames/s", "n_gpus": world,
                          "dry_run": True, "config": {"workload": args.config},
                          "slabs": slab_ranges(cfg.dims, world)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--only", action="store_true", help="measure only --config (no other_configs)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=120.0)
    ap.add_argument("--dry-run", action="store_true")
    ap.add_argument("--pipeline", action="store_true", help="c1/c5: the end-to-end multilevel run")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one rank per GPU: re-launch under torchrun (the driver launches torchrun itself; this is for
        # a plain `python bench.py --gpus N`)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.dry_run:
        run_dry(args)
    elif args.pipeline:
        run_pipeline(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
