"""Diagnostic: fused vs unfused curvature gradient and run-to-run determinism on a small 2-D NGF problem."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_2001_06613_b200 as srb  # noqa: E402
from test_parity_gpu import _frames_dev, _random_problem  # noqa: E402

dims = (40, 24)
rng = np.random.default_rng(5)
frames, spacing, origin, y, w = _random_problem(rng, dims, 5, amp=0.3)
print("spacing", spacing, "origin", origin)
h = float(np.prod(spacing))
fd = _frames_dev(frames, dims, spacing, origin, torch.float32)
yt = torch.as_tensor(y).to(device=fd.data.device, dtype=torch.float32).contiguous()
obj = srb.FieldObjective(fd, list(range(5)), w, h, feature="ngf", ngf_eps=0.5, alpha=1.5)
plan = obj.plan
prob = plan.problem(y=yt)
gs = []
for i in range(3):
    g2 = torch.empty_like(yt)
    plan.evaluate(prob, w, h, g2)
    gs.append(g2.clone())
print("plan.evaluate run-to-run equal:", torch.equal(gs[0], gs[1]), torch.equal(gs[1], gs[2]))
stats, g = obj.evaluate(yt)
g = g.clone()
s2 = torch.zeros(1, dtype=torch.float64, device=yt.device)
g2 = gs[0].clone()
plan.curvature(prob, 1.5, h, g2, s2)
dd = (g - g2).abs()
print("fused vs unfused max diff", float(dd.max()), "max |g|", float(g.abs().max()), "n diff", int((dd > 0).sum()), "of", dd.numel())
idx = torch.nonzero(dd > 0)
print(idx[:20].tolist())
