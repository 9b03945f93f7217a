"""Every kernel variant selectable by environment switch (read once per engine context) gives the
oracle's D and dD/dy: each variant runs the fp32 field parity cases in a fresh process.

    SEQREG_B200_LEGACY=1  non-specialized pass 1 / pass 2 (the generic kernels)
    SEQREG_B200_TC=0      no tensor-core split pass 1: warp-specialized SIMT Gram (k_pass1_ws) for NCC,
                          the generic NGF kernels
    SEQREG_B200_P2S=0     re-gathering pass 2 (default: streaming pass 2 from the split pass 1's V, grad T)
    SEQREG_B200_GRAPH=0   no CUDA-graph replay of repeated sr_evaluate calls
    SEQREG_B200_P2TMA=0   2-D NCC pass 2 loads straight from HBM (k_pass2_mma; default TMA-fed k_pass2_tma)
    SEQREG_B200_SFEAT=0   2-D NGF: the generic fused sampler k_ngf_sfeat2 instead of k_ngf_sfeat2f

(The round-1 variants measured slower — tcgen05 NCC pass 1 / pass 2, warp-specialized pass 2, fused
sampling + Gram, texture gathers, PDL, the unpipelined sampler — were removed from the library.)
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np, torch
import paper_2001_06613_b200 as srb
from oracle import seqreg_oracle as orc
from scipy.ndimage import gaussian_filter

out = []
for feature, dims, K, seed in [("ncc", (64, 48), 32, 1), ("ncc", (40, 36), 20, 2), ("ncc", (200, 150), 32, 3),
                               ("ncc", (12, 11, 10), 32, 4), ("ngf", (64, 48), 32, 5), ("ngf", (40, 36), 60, 6),
                               ("ngf", (12, 11, 10), 20, 7)]:
    rng = np.random.default_rng(seed)
    d = len(dims)
    sp = tuple([0.5, 0.25, 0.75][:d])
    org = tuple(-n * s / 2 for n, s in zip(dims, sp))
    frames = np.stack([gaussian_filter(rng.standard_normal(dims), 1.5, mode="reflect").ravel(order="F") + 3.0
                       for _ in range(K)])
    x = orc.cell_centers(dims, sp, org).T
    y = x[None] + 0.4 * rng.standard_normal((K,) + x.shape) * np.asarray(sp)[None, :, None]
    # keep samples off grid nodes, where the interpolant's derivative jumps and an fp32 rounding of y
    # flips the cell (the kink hazard; covered separately by the dyadic identity test)
    s_ = np.asarray(sp)[None, :, None]
    o_ = np.asarray(org)[None, :, None]
    t_ = (y - o_) / s_ - 0.5
    fr = t_ - np.floor(t_)
    y = np.where((fr < 2e-3) | (fr > 1 - 2e-3), y + 5e-3 * s_, y)
    w = rng.uniform(0.5, 1.0, K)
    h = float(np.prod(sp))
    fd = srb.DeviceFrames.from_array(srb.get_engine(), frames, srb.GridSpec(dims, sp, org), torch.float32)
    obj = srb.FieldObjective(fd, list(range(K)), w, h, feature=feature, ngf_eps=0.2)
    yt = torch.as_tensor(y).to(device=fd.data.device, dtype=torch.float32).contiguous()
    stats, g = obj.evaluate(yt)
    D = float(stats[0].item())
    q = frames.astype(np.float32).astype(np.float64)
    yq = y.astype(np.float32).astype(np.float64)
    _, Dref, gref = orc.evaluate_field(list(q), dims, sp, org, yq, w, h, feature, 0.2)
    gd = g.double().cpu().numpy()
    out.append({"feature": feature, "dims": list(dims), "K": K, "dD": abs(D - Dref) / abs(Dref),
                "dg": float(np.abs(gd - gref).max() / np.abs(gref).max())})
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", ["SEQREG_B200_LEGACY=1", "SEQREG_B200_TC=0", "SEQREG_B200_P2S=0", "SEQREG_B200_GRAPH=0",
                                 "SEQREG_B200_P2TMA=0", "SEQREG_B200_SFEAT=0", ""])
def test_variant_parity(env):
    e = dict(os.environ)
    if env:
        k, v = env.split("=")
        e[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    for case in json.loads(r.stdout.strip().splitlines()[-1]):
        assert case["dD"] < 1e-4 and case["dg"] < 1e-4, (env, case)
