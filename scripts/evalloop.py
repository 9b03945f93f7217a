"""A few fused evaluations (L2 flushed in between) of a bench config, for profilers:

    ncu --metrics gpu__time_duration.sum -k regex:"k_" python scripts/evalloop.py --reps 3
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
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--finalize-only", action="store_true", help="loop sr_corr_finalize on one pass-1 result")
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
    flush_w = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    flush_r = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    if args.finalize_only:
        plan.corr_partial(prob)
    for i in range(args.reps):
        flush_w.fill_(float(i))
        flush_r.sum()
        if args.finalize_only:
            plan.finalize(prob, w, grid.cell_volume)
        else:
            plan.evaluate(prob, w, grid.cell_volume, g)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
