"""NGF pass-1 / pass-2 time vs K at 1024^2 fp32 (how the work splits between the per-sample
feature work, linear in K, and the K x K Gram, quadratic in K).

    python scripts/ngf_k_sweep.py
"""

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2001_06613_b200 as srb  # noqa: E402
from paper_2001_06613_b200 import synth  # noqa: E402


def main():
    cfg = synth.CONFIGS["c3"]
    out = {}
    for K in (8, 16, 32, 64, 100, 128):
        frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device="cuda", K=K)
        y = synth.smooth_noise_iterate(cfg.dims, K, device="cuda").to(torch.float32).contiguous()
        grid = srb.GridSpec(cfg.dims, spacing, origin)
        fd = srb.DeviceFrames(srb.get_engine(), frames.to(torch.float32), grid)
        plan = srb.EvalPlan(fd, list(range(K)), feature="ngf", ngf_eps=cfg.ngf_eps)
        prob = plan.problem(y=y)
        g = torch.empty_like(y)
        w = np.full(K, 1.0 / K)
        for _ in range(2):
            plan.evaluate(prob, w, grid.cell_volume, g)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        reps = 3
        t = np.zeros(3)
        for _ in range(reps):
            ev[0].record()
            plan.corr_partial(prob)
            ev[1].record()
            plan.finalize(prob, w, grid.cell_volume)
            ev[2].record()
            plan.grad(prob, g)
            ev[3].record()
            torch.cuda.synchronize()
            t += [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])]
        out[K] = (t / reps).round(3).tolist()
        print(K, out[K], flush=True)
        del fd, plan, frames, y, g
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
