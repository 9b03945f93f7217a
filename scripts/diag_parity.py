"""Diagnostic (GPU box): full-size gradient error map of the CUDA path against the CPU oracle.

    python scripts/diag_parity.py c3 [--oracle /tmp/c3_oracle.npz] [--dtype f32|f64]

Computes (or loads) the oracle's D, C and full dD/dy for the config's seeded inputs (fp64 arithmetic on
the float32-quantised inputs, exactly tests/golden/make_config_golden.py), evaluates the CUDA path, and
prints where the gradient differs: per frame (norm and max), per slowest-axis row band, boundary vs
interior.  Test infrastructure only (imports the oracle as the checker).
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("--oracle", default=None)
    ap.add_argument("--dtype", default="f32")
    args = ap.parse_args()
    import make_config_golden as mk

    from oracle import seqreg_oracle as orc

    fr, yv, w, spacing, origin, cfg = mk.config_inputs(args.name)
    K, d, N = yv.shape
    h = float(np.prod(spacing))
    path = Path(args.oracle or f"/tmp/{args.name}_oracle.npz")
    if path.exists():
        z = np.load(path)
        Dref, Cref, gref = float(z["D"]), z["C"], z["g"]
    else:
        t0 = time.time()
        st, Dref, gref = orc.evaluate_field(list(fr), cfg.dims, spacing, origin, yv, w, h, cfg.feature,
                                            cfg.ngf_eps, threads=os.cpu_count() or 8)
        Cref = st.corr
        np.savez(path, D=Dref, C=Cref, g=gref)
        print(f"oracle {time.time() - t0:.1f} s", flush=True)

    import paper_2001_06613_b200 as srb

    dt = torch.float32 if args.dtype == "f32" else torch.float64
    dev = torch.device("cuda", 0)
    eng = srb.get_engine(0)
    fd = srb.DeviceFrames(eng, torch.as_tensor(fr, dtype=dt).to(dev), srb.GridSpec(cfg.dims, spacing, origin))
    y = torch.as_tensor(yv, dtype=dt).to(dev).contiguous()
    obj = srb.FieldObjective(fd, list(range(K)), w, h, feature=cfg.feature, ngf_eps=cfg.ngf_eps)
    stats, g = obj.evaluate(y)
    torch.cuda.synchronize()
    hs = obj.host_stats()
    g = g.double().cpu().numpy()
    gmax = np.abs(gref).max()
    err = np.abs(g - gref) / gmax
    print(f"{args.name} {args.dtype} env={ {k: v for k, v in os.environ.items() if k.startswith('SEQREG')} }")
    print(f"D {hs['D']:.12g} ref {Dref:.12g} rel {abs(hs['D'] - Dref) / abs(Dref):.2e}; "
          f"C max abs err {np.abs(hs['corr'] - Cref).max():.2e}")
    print(f"grad max err/gmax {err.max():.3e} mean {err.mean():.3e}")
    gn = np.sqrt((g.reshape(K, -1) ** 2).sum(1))
    gnr = np.sqrt((gref.reshape(K, -1) ** 2).sum(1))
    en = np.abs(gn - gnr) / gnr.max()
    print("per-frame norm err/max: worst", np.argsort(-en)[:8], en[np.argsort(-en)[:8]])
    print("per-frame rel norm err (gn/gnr-1):", np.round((gn / gnr - 1) * 1e4, 2).tolist(), "x1e-4")
    ef = err.reshape(K, -1).max(1)
    print("per-frame max err:", np.round(ef * 1e5, 2).tolist(), "x1e-5")
    grid = err.max(axis=(0, 1)).reshape(tuple(reversed(cfg.dims)))  # [slow..fast]
    slow = grid.reshape(grid.shape[0], -1).max(1)
    print("max err by slowest-axis index (first 4, last 4, worst 8):", slow[:4], slow[-4:],
          np.argsort(-slow)[:8], slow[np.argsort(-slow)[:8]])
    fast = grid.reshape(-1, grid.shape[-1]).max(0)
    print("max err by fastest-axis index (first 4, last 4, worst 8):", fast[:4], fast[-4:],
          np.argsort(-fast)[:8], fast[np.argsort(-fast)[:8]])
    # difference pattern: is the error proportional to the gradient (a scale error per frame)?
    for k in np.argsort(-en)[:3]:
        a, b = g[k].ravel(), gref[k].ravel()
        s = float(a @ b / (b @ b))
        r = a - s * b
        print(f"frame {k}: best scale {s:.8f}; residual after scale max {np.abs(r).max() / gmax:.2e}")


if __name__ == "__main__":
    main()
