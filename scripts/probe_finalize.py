"""Time the reduce / finalize stages alone at a bench config (CUDA events, back to back, no flush).

    python scripts/probe_finalize.py [--config c2] [--reps 200]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2001_06613_b200 as srb  # noqa: E402
from paper_2001_06613_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=200)
    args = ap.parse_args()
    cfg = synth.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device=dev)
    y = synth.smooth_noise_iterate(cfg.dims, cfg.K, device=dev).to(cfg.dtype).contiguous()
    eng = srb.get_engine(0)
    grid = srb.GridSpec(cfg.dims, spacing, origin)
    fd = srb.DeviceFrames(eng, frames.to(cfg.dtype), grid)
    w = synth.config_weights(cfg)
    plan = srb.EvalPlan(fd, list(range(cfg.K)), feature=cfg.feature, ngf_eps=cfg.ngf_eps)
    prob = plan.problem(y=y)
    g = torch.empty_like(y)
    st = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(10):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(args.reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.reps * 1e3

    plan.corr_partial(prob)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof0:
        for _ in range(20):
            plan.corr_partial(prob)  # reduce only (no finalize)
        torch.cuda.synchronize()
    for ev in prof0.events():
        if ev.device_type.name == "CUDA" and "reduce" in ev.name:
            print(f"  reduce only: {ev.name.split('(')[0][-40:]} {ev.device_time:.2f} us")
            break
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(20):
            plan.finalize(prob, w, grid.cell_volume)
        for _ in range(20):
            plan.evaluate(prob, w, grid.cell_volume, g)
        torch.cuda.synchronize()
    acc = {}
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            n = ev.name.split("(")[0][-40:]
            acc.setdefault(n, []).append(ev.device_time)
    for n, v in sorted(acc.items()):
        print(f"  {n:42s} n={len(v):3d} mean {sum(v) / len(v):8.2f} us")
    print(f"finalize only (k_finalize): {timed(lambda: plan.finalize(prob, w, grid.cell_volume)):.2f} us")
    print(f"corr_partial (pass 1 + reduce): {timed(lambda: plan.corr_partial(prob)):.2f} us")
    print(f"evaluate: {timed(lambda: plan.evaluate(prob, w, grid.cell_volume, g)):.2f} us")
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.reps):
        plan.evaluate(prob, w, grid.cell_volume, g)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"host enqueue per evaluate: {(t1 - t0) / args.reps * 1e6:.2f} us")
    gr = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream()
    with torch.cuda.stream(s2):
        plan.evaluate(prob, w, grid.cell_volume, g)
        torch.cuda.synchronize()
        with torch.cuda.graph(gr, stream=s2):
            plan.evaluate(prob, w, grid.cell_volume, g)
    torch.cuda.synchronize()
    print(f"graph replay: {timed(lambda: gr.replay()):.2f} us")


if __name__ == "__main__":
    main()
