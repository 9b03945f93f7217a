"""Device L-BFGS (sr_lbfgs_minimize) at the C5 parameter size, beside the numpy oracle L-BFGS.

n = K * d * N = 64 * 2 * 1024^2 fp64 parameters (537 MB in fp32, 1.07 GB in fp64).
The objective is a separable quadratic f = 0.5 sum d_i x_i^2 - b.x evaluated on the device
(2 passes), so the optimizer's own vector algebra dominates.  Bytes per iteration of the device
algebra (fp64, history L = memory once full): q = g (16), L x [dot(s, q) 16 + axpy 24], scale 16,
L x [dot(y, q) 16 + axpy 24], negate 16, g.p 16, x + step p 24, s = xn - x 24, y = gn - g 24,
s.y / s.s / y.y / |g| 56, x <- xn 16  =>  232 + 80 L  bytes per parameter (L = pairs in the history),
averaged over the iterations actually run.

    python scripts/bench_lbfgs.py [--n N] [--iters 10] [--cpu-iters 2] > profiles/r01_lbfgs.json
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2001_06613_b200.optimizer import ObjectiveEval, OptimOptions, lbfgs_minimize  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64 * 2 * 1024 * 1024)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--cpu-iters", type=int, default=2)
    ap.add_argument("--cpu-n", type=int, default=0, help="oracle size (default: the same n)")
    a = ap.parse_args()
    n = a.n
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    dvec = torch.rand(n, generator=g, device=dev, dtype=torch.float64) * 9.0 + 1.0
    bvec = torch.randn(n, generator=g, device=dev, dtype=torch.float64)
    obj_time = [0.0]

    def obj(x):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        m = x.numel()
        dx = dvec[:m] * x
        f = 0.5 * torch.dot(x, dx) - torch.dot(bvec[:m], x)
        gr = dx - bvec[:m]
        e1.record()
        torch.cuda.synchronize()
        obj_time[0] += e0.elapsed_time(e1) * 1e-3
        return ObjectiveEval(float(f.item()), gr)

    opts = OptimOptions(max_iters=a.iters, grad_tol=1e-30, f_tol=1e-30, step_tol=1e-30)
    x0 = torch.zeros(n, dtype=torch.float64, device=dev)
    lbfgs_minimize(obj, x0.clone(), OptimOptions(max_iters=1))  # warm-up at full size (workspace, kernels)
    torch.cuda.synchronize()
    obj_time[0] = 0.0
    t0 = time.perf_counter()
    res = lbfgs_minimize(obj, x0, opts)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    algebra = wall - obj_time[0]
    it = max(res.iterations, 1)
    # history length L_i = min(i - 1, memory) on iteration i (no curvature pair is rejected on this
    # convex problem); every extra backtracking trial re-forms x + step p (24 B per parameter)
    total = sum(232 + 80 * min(i - 1, opts.memory) for i in range(1, res.iterations + 1))
    total += 24 * max(0, res.objective_evaluations - 1 - res.iterations)
    bytes_per_iter = total * n / it
    peak = 6549.1
    try:
        peak = float(json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        pass
    line = {
        "metric": "device L-BFGS vector algebra per iteration (C5 parameter size)",
        "n": n, "iterations": res.iterations, "evaluations": res.objective_evaluations,
        "reason": res.converged_reason,
        "ms_per_iteration_algebra": algebra / it * 1e3, "ms_per_iteration_objective": obj_time[0] / it * 1e3,
        "bytes_per_iteration_algebra": bytes_per_iter,
        "achieved_gbs": bytes_per_iter / (algebra / it) / 1e9, "peak_gbs": peak,
        "frac": bytes_per_iter / (algebra / it) / 1e9 / peak,
    }
    # ---- the numpy oracle L-BFGS on the host (bounded), same objective restated in numpy
    if a.cpu_iters > 0:
        from oracle import seqreg_oracle as orc

        cn = a.cpu_n or n
        dh = dvec[:cn].cpu().numpy()
        bh = bvec[:cn].cpu().numpy()

        def hobj(x):
            dx = dh * x
            return 0.5 * x @ dx - bh @ x, dx - bh

        t0 = time.perf_counter()
        r = orc.lbfgs_minimize(hobj, np.zeros(cn), max_iters=a.cpu_iters, grad_tol=1e-30, f_tol=1e-30, step_tol=1e-30)
        cw = time.perf_counter() - t0
        line["cpu_oracle"] = {"n": cn, "iterations": r["iterations"], "s_per_iteration_total": cw / max(r["iterations"], 1),
                              "cores": 1, "kind": "port"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
