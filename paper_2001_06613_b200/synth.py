"""Seeded synthetic sequences for the BASELINE.json configurations.

The reference's own generator (synth.py:55-124) makes 2-D affine sequences only;
the BASELINE configs need Gaussian-blob images warped by smooth sinusoidal
motion, written fresh here.  Draw order from
``numpy.random.default_rng(seed)``: blob centres, sigmas, amplitudes, then the
per-frame noise.  Images are evaluated analytically (no interpolation bias):

    R(x)   = sum_b a_b exp(-|x - c_b|^2 / (2 s_b^2))
    T_k(x) = R(x + u(x, t_k)) + noise,  t_k = (k-1)/(K-1)

Evaluation runs in float64 on any torch device (CUDA for the large configs).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

__all__ = ["SeqConfig", "CONFIGS", "make_sequence", "cell_centers", "smooth_noise_iterate", "config_weights",
           "bench_iterate"]


@dataclass(frozen=True)
class SeqConfig:
    name: str
    dims: tuple
    K: int
    n_blobs: int
    amp: float           # motion amplitude
    cycles: float        # temporal cycles of the motion over t in [0, 1]
    noise: float         # noise standard deviation
    feature: str
    ngf_eps: float
    weights: str         # "uniform" | "uniform_random" (U[0.5, 1])
    dtype: torch.dtype
    alpha: float = 0.0   # curvature regulariser weight
    sigma_range: tuple = (0.03, 0.1)
    amp_range: tuple = (0.5, 1.0)


# BASELINE.json "configs" restated.
CONFIGS = {
    "c1": SeqConfig("c1", (128, 128), 10, 8, 0.05, 1.0, 0.01, "ngf", 0.1, "uniform", torch.float64, alpha=1.0),
    "c2": SeqConfig("c2", (512, 512), 32, 24, 0.08, 1.0, 0.01, "ncc", 0.1, "uniform_random", torch.float32),
    "c3": SeqConfig("c3", (1024, 1024), 100, 64, 0.06, 2.0, 0.02, "ngf", 0.05, "uniform", torch.float32),
    "c4": SeqConfig("c4", (128, 128, 128), 20, 32, 0.04, 1.0, 0.01, "ngf", 0.1, "uniform", torch.float32),
    "c5": SeqConfig("c5", (1024, 1024), 64, 24, 0.05, 1.0, 0.01, "ngf", 0.1, "uniform", torch.float32, alpha=10.0),
}


def cell_centers(dims, spacing=None, origin=None, device="cpu") -> torch.Tensor:
    """[d, N] cell centres, first axis fastest (grid.py:170-187)."""
    d = len(dims)
    spacing = spacing or tuple(1.0 / n for n in dims)
    origin = origin or (0.0,) * d
    axes = [origin[a] + (torch.arange(dims[a], dtype=torch.float64, device=device) + 0.5) * spacing[a]
            for a in range(d)]
    mesh = torch.meshgrid(*axes, indexing="ij")
    # ravel(order="F"): first axis fastest == permute to reversed axes then flatten C-order
    return torch.stack([m.permute(*reversed(range(d))).reshape(-1) for m in mesh])


def _motion(x: torch.Tensor, t: float, amp: float, cycles: float) -> torch.Tensor:
    """u(x, t) = amp sin(2 pi cycles t) * pattern(x); 2-D pattern [sin sin, cos sin] (BASELINE.json),
    3-D pattern [sin sin sin, cos sin sin, sin cos sin]."""
    d = x.shape[0]
    s = torch.sin(math.pi * x)
    c = torch.cos(math.pi * x)
    if d == 2:
        pat = torch.stack([s[0] * s[1], c[0] * s[1]])
    else:
        pat = torch.stack([s[0] * s[1] * s[2], c[0] * s[1] * s[2], s[0] * c[1] * s[2]])
    return amp * math.sin(2.0 * math.pi * cycles * t) * pat


def make_sequence(cfg: SeqConfig, seed: int = 0, device="cpu", K: int | None = None, dims=None):
    """Returns (frames [K, N] float64 tensor on ``device``, times (K,), spacing, origin)."""
    dims = tuple(dims or cfg.dims)
    K = int(K or cfg.K)
    d = len(dims)
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, 1.0, size=(cfg.n_blobs, d))
    sig = rng.uniform(*cfg.sigma_range, size=cfg.n_blobs)
    amps = rng.uniform(*cfg.amp_range, size=cfg.n_blobs)
    spacing = tuple(1.0 / n for n in dims)
    origin = (0.0,) * d
    x = cell_centers(dims, spacing, origin, device)
    N = x.shape[1]
    times = np.array([(k / (K - 1)) for k in range(K)]) if K > 1 else np.zeros(1)
    frames = torch.empty((K, N), dtype=torch.float64, device=device)
    cen = torch.as_tensor(centres, device=device)
    sg = torch.as_tensor(sig, device=device)
    am = torch.as_tensor(amps, device=device)
    for k in range(K):
        p = x + _motion(x, float(times[k]), cfg.amp, cfg.cycles)
        acc = torch.zeros(N, dtype=torch.float64, device=device)
        for b in range(cfg.n_blobs):
            r2 = ((p - cen[b][:, None]) ** 2).sum(0)
            acc += am[b] * torch.exp(-r2 / (2.0 * sg[b] ** 2))
        noise = rng.standard_normal(N) * cfg.noise
        frames[k] = acc + torch.as_tensor(noise, device=device)
    return frames, times, spacing, origin


def _gauss_kernel(sigma_px: float, device) -> torch.Tensor:
    r = int(math.ceil(4.0 * sigma_px))
    t = torch.arange(-r, r + 1, dtype=torch.float64, device=device)
    k = torch.exp(-0.5 * (t / sigma_px) ** 2)
    return k / k.sum()


def _smooth_axis(a: torch.Tensor, kern: torch.Tensor, axis: int) -> torch.Tensor:
    """Separable convolution along ``axis`` of an nd array with reflect padding."""
    r = (kern.numel() - 1) // 2
    moved = a.movedim(axis, -1)
    shp = moved.shape
    flat = moved.reshape(-1, 1, shp[-1])
    pad = torch.nn.functional.pad(flat, (r, r), mode="reflect")
    out = torch.nn.functional.conv1d(pad, kern.view(1, 1, -1))
    return out.reshape(shp).movedim(-1, axis)


def smooth_noise_iterate(dims, K: int, sigma_px: float = 4.0, std_px: float = 0.5, seed: int = 1,
                         device="cpu") -> torch.Tensor:
    """Config-2 iterate y = x + G_sigma * N(0, std) per component, in world units: [K, d, N] float64."""
    d = len(dims)
    rng = np.random.default_rng(seed)
    spacing = tuple(1.0 / n for n in dims)
    x = cell_centers(dims, spacing, None, device)
    kern = _gauss_kernel(sigma_px, device)
    out = torch.empty((K, d, x.shape[1]), dtype=torch.float64, device=device)
    for k in range(K):
        for c in range(d):
            z = torch.as_tensor(rng.standard_normal(tuple(reversed(dims))), device=device)  # C-order of F-raveled
            for ax in range(d):
                z = _smooth_axis(z, kern, ax)
            out[k, c] = x[c] + z.reshape(-1) * std_px * spacing[c]
    return out


def config_weights(cfg: SeqConfig, K: int | None = None, seed: int = 2) -> np.ndarray:
    K = int(K or cfg.K)
    if cfg.weights == "uniform_random":
        return np.random.default_rng(seed).uniform(0.5, 1.0, size=K)
    return np.full(K, 1.0 / K)


def bench_iterate(cfg: SeqConfig, device="cpu", dims=None) -> torch.Tensor:
    """The displacement iterate every arm of bench.py and the config goldens evaluate at: BASELINE
    configs[1]'s recipe y = x + G_(sigma=4 px) * N(0, 0.5 px) per component (seed 1), applied to every
    config so the GPU arm, the CPU baseline, the reference arm and tests/golden/config_golden.npz see the
    same iterate.  [K, d, N] float64 (cast to the config dtype by the caller)."""
    return smooth_noise_iterate(tuple(dims or cfg.dims), cfg.K, sigma_px=4.0, std_px=0.5, seed=1, device=device)
