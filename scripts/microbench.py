"""Kernel A/B timings for the C2 workload (pass 1 / pass 2 split), CUDA events, L2 flushed.

    python scripts/microbench.py [--config c2] [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2001_06613_b200 as srb  # noqa: E402
from paper_2001_06613_b200 import synth  # noqa: E402


def timeit(fn, flush, reps):
    st = torch.cuda.current_stream()
    ts = []
    for i in range(reps + 3):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts)) * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device=dev)
    y = synth.smooth_noise_iterate(cfg.dims, cfg.K, device=dev).to(cfg.dtype).contiguous()
    eng = srb.get_engine(0)
    grid = srb.GridSpec(cfg.dims, spacing, origin)
    fd = srb.DeviceFrames(eng, frames.to(cfg.dtype), grid)
    w = synth.config_weights(cfg)
    K, N = cfg.K, grid.cell_count
    flush_w = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    flush_r = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    class Flush:  # write 256 MiB then read 256 MiB: L2 ends up holding clean, unrelated lines
        def fill_(self, v):
            flush_w.fill_(v)
            flush_r.sum()

    flush = Flush()
    res = {}
    plan = srb.EvalPlan(fd, list(range(K)), feature=cfg.feature, ngf_eps=cfg.ngf_eps)
    prob = plan.problem(y=y)
    g = torch.empty_like(y)
    # padded copy of y: stride N + 1 disables the TMA / 16-byte paths
    ypad = torch.zeros((K, len(cfg.dims), N + 1), dtype=y.dtype, device=dev)
    ypad[..., :N] = y
    prob_pad = plan.problem(y=ypad)
    prob = plan.problem(y=y)
    for ctas in [0, 148, 296, 444, 592]:
        eng.set_grid_ctas(ctas)
        res[f"pass1 ctas={ctas}"] = timeit(lambda: plan.corr_partial(prob), flush, args.reps)
    eng.set_grid_ctas(0)

    class NoFlush:
        def fill_(self, v):
            pass

    res["pass1 warm L2 (no flush)"] = timeit(lambda: plan.corr_partial(prob), NoFlush(), args.reps)
    res["pass2 warm L2 (no flush)"] = timeit(lambda: plan.grad(prob, g), NoFlush(), args.reps)
    fr_only = fd.data

    class FramesHot:  # flush, then pull the frames (33.5 MB) back into L2
        def fill_(self, v):
            flush.fill_(v)
            fr_only.sum()

    res["pass1 frames in L2, y cold"] = timeit(lambda: plan.corr_partial(prob), FramesHot(), args.reps)
    res["pass2 frames in L2, y cold"] = timeit(lambda: plan.grad(prob, g), FramesHot(), args.reps)
    prob_pad = plan.problem(y=ypad)
    res["pass1 y-stride N+1 (no TMA/vec)"] = timeit(lambda: plan.corr_partial(prob_pad), flush, args.reps)
    prob = plan.problem(y=y)
    plan.corr_partial(prob)
    plan.finalize(prob, w, grid.cell_volume)
    res["finalize"] = timeit(lambda: plan.finalize(prob, w, grid.cell_volume), flush, args.reps)
    for ctas in [0, 148, 296, 592, 888]:
        eng.set_grid_ctas(ctas)
        res[f"pass2 ctas={ctas}"] = timeit(lambda: plan.grad(prob, g), flush, args.reps)
    eng.set_grid_ctas(0)
    res["evaluate (fused entry)"] = timeit(lambda: plan.evaluate(prob, w, grid.cell_volume, g), flush, args.reps)
    # a pure streaming reference on the same device: read y + frames once
    z = torch.zeros(1, device=dev)
    res["trivial kernel (event overhead)"] = timeit(lambda: z.add_(1.0), flush, args.reps)
    yc = torch.empty_like(y)
    res["torch copy y (67MB read + 67MB write)"] = timeit(lambda: yc.copy_(y), flush, args.reps)
    res["torch y.sum()+frames.sum() (read 100MB)"] = timeit(lambda: (y.sum(), fd.data.sum()), flush, args.reps)
    # per-kernel device durations (CUPTI) of 10 fused evaluations, L2 flushed in between
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(10):
            flush.fill_(float(i))
            plan.evaluate(prob, w, grid.cell_volume, g)
        torch.cuda.synchronize()
    kt = {}
    for ev in prof.events():
        if ev.device_type.name == "CUDA" and "sr::" in ev.name:
            key = ev.name.split("(")[0].replace("void sr::", "").replace("sr::", "")[:60]
            kt.setdefault(key, []).append(ev.device_time)
    for k2, v in kt.items():
        res["kernel " + k2] = float(np.mean(v))
    print(json.dumps({"legacy": os.environ.get("SEQREG_B200_LEGACY", "0"), **{k: round(v, 1) for k, v in res.items()}},
                     indent=1))


if __name__ == "__main__":
    main()
