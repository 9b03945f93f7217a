"""Small evaluations through every default kernel family, for compute-sanitizer (tests/test_sanitizer_gpu.py):
fp32 NCC K = 24 (k_sample_vp, k_gram_tma, k_reduce_finalize, k_pass2_tma), fp32 NGF K = 40 and K = 100
(k_ngf_sfeat2f, k_gram_h<64|128>, k_ngf_z_tc), fp32 NGF K = 20 (k_gram_h<32>, k_ngf_z_f16), 3-D fp32 NGF,
fp64 NGF (generic kernels), the fused curvature (sr_evaluate_reg) and a 129-frame subset (frame blocks)."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2001_06613_b200 as srb  # noqa: E402


def case(dims, K, feature, dtype, alpha=0.0, seed=0):
    from scipy.ndimage import gaussian_filter

    rng = np.random.default_rng(seed)
    sp = tuple(1.0 / n for n in dims)
    org = (0.0,) * len(dims)
    frames = np.stack([gaussian_filter(rng.standard_normal(dims), 1.5).ravel(order="F") + 2.0 for _ in range(K)])
    axes = [(np.arange(n) + 0.5) / n for n in dims]
    x = np.stack([m.ravel(order="F") for m in np.meshgrid(*axes, indexing="ij")])
    y = x[None] + 0.3 * rng.standard_normal((K,) + x.shape) * np.asarray(sp)[None, :, None]
    eng = srb.get_engine(0)
    fd = srb.DeviceFrames.from_array(eng, frames, srb.GridSpec(dims, sp, org), dtype)
    obj = srb.FieldObjective(fd, list(range(K)), rng.uniform(0.5, 1, K), feature=feature, ngf_eps=0.3, alpha=alpha)
    yt = torch.as_tensor(y, dtype=dtype, device="cuda:0").contiguous()
    for _ in range(2):
        stats, g = obj.evaluate(yt)
    torch.cuda.synchronize()
    assert np.isfinite(float(stats[0].item())) and bool(torch.isfinite(g).all())


def main():
    case((64, 48), 24, "ncc", torch.float32)
    case((64, 48), 40, "ngf", torch.float32)
    case((64, 48), 100, "ngf", torch.float32, alpha=1.0)
    case((64, 48), 20, "ngf", torch.float32)
    case((16, 12, 10), 12, "ngf", torch.float32)
    case((24, 20), 6, "ngf", torch.float64, alpha=1.0)
    case((16, 12), 129, "ncc", torch.float64)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
