"""GPU pyramid (sr_pyramid_step) and field prolongation (sr_prolong_field) at the C5 shape, beside
the numpy oracle on a bounded sample.

Compulsory bytes: a pyramid step over F frames of N cells reads the stack once and writes N/2^d
per frame (smoothing and restriction are fused in registers); prolongation reads k d N_c and writes
k d N_f values.  Kernel times are CUPTI device times (torch.profiler).

    python scripts/bench_spatial.py > profiles/r01_spatial_c5.json
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2001_06613_b200 as srb  # noqa: E402
from paper_2001_06613_b200 import synth  # noqa: E402


def _peak():
    try:
        return float(json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6549.1


def main():
    dims, F, levels, s = (1024, 1024), 64, 4, 4
    grid = srb.GridSpec(dims, (1 / 1024, 1 / 1024), (0.0, 0.0))
    data = torch.randn((F, grid.cell_count), device="cuda", dtype=torch.float32)
    fd = srb.DeviceFrames(srb.get_engine(), data, grid)
    from torch.profiler import ProfilerActivity, profile

    N = grid.cell_count
    k = 64
    srb.build_pyramid(fd, levels)
    step = srb.pyramid_step(fd)
    cg = step.grid
    yc = synth.cell_centers(cg.dims, cg.spacing, cg.origin, device="cuda").to(torch.float32).unsqueeze(0).repeat(k, 1, 1)
    yc = yc.contiguous()
    srb.prolong_field(yc, cg, grid)
    torch.cuda.synchronize()
    reps = 5
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            srb.pyramid_step(fd)
            srb.prolong_field(yc, cg, grid)
        torch.cuda.synchronize()
    kt = {}
    for ev in prof.events():
        if ev.device_type.name == "CUDA" and "sr::" in ev.name:
            key = "pyramid" if "k_pyramid" in ev.name else ("prolong" if "k_prolong_field" in ev.name else None)
            if key:
                kt.setdefault(key, []).append(ev.device_time)
    ms_step = float(np.mean(kt["pyramid"])) * 1e-3
    ms_prol = float(np.mean(kt["prolong"])) * 1e-3
    bytes_step = (s * N + s * N // 4) * F
    t0 = time.perf_counter()
    pyr = srb.build_pyramid(fd, levels)
    torch.cuda.synchronize()
    ms_build = (time.perf_counter() - t0) * 1e3
    bytes_prol = s * k * 2 * (cg.cell_count + N)
    # numpy oracle on one frame (bounded), scaled to the F frames
    from oracle import seqreg_oracle as orc

    one = data[0].double().cpu().numpy()
    t0 = time.perf_counter()
    orc.pyramid_step_flat(one, dims)
    cpu_frame = time.perf_counter() - t0
    peak = _peak()
    print(json.dumps({
        "metric": "GPU pyramid step and field prolongation at the C5 shape (1024^2, 64 frames, fp32)",
        "pyramid_step_ms": ms_step, "pyramid_step_bytes": bytes_step,
        "pyramid_step_gbs": bytes_step / (ms_step * 1e-3) / 1e9, "pyramid_step_frac": bytes_step / (ms_step * 1e-3) / 1e9 / peak,
        "build_pyramid_4_levels_ms_wall": ms_build, "timing": "CUPTI kernel device time, mean of 5", "levels": [list(p.grid.dims) for p in pyr],
        "prolong_ms": ms_prol, "prolong_bytes": bytes_prol,
        "prolong_gbs": bytes_prol / (ms_prol * 1e-3) / 1e9, "prolong_frac": bytes_prol / (ms_prol * 1e-3) / 1e9 / peak,
        "peak_gbs": peak,
        "cpu_oracle": {"kind": "port", "cores": 1, "sample": "one 1024^2 frame, numpy restatement of pyramid.py",
                       "s_per_frame": cpu_frame, "s_per_step_scaled": cpu_frame * F},
    }))


if __name__ == "__main__":
    main()
