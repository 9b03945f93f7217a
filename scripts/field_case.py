"""One small fp32 NCC displacement evaluation vs the oracle (debug helper for kernel variants;
samples are not kept off grid nodes, so fp32 kink flips can show up in dg).

    SEQREG_B200_<SWITCH>=1 python scripts/field_case.py n0 n1 K
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2001_06613_b200 as srb  # noqa: E402
from oracle import seqreg_oracle as orc  # noqa: E402

dims = tuple(int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (64, 48)))
K = int(sys.argv[3]) if len(sys.argv) > 3 else 32
rng = np.random.default_rng(1)
sp = (1.0 / dims[0], 1.0 / dims[1])
org = (0.0, 0.0)
frames = rng.standard_normal((K, dims[0] * dims[1])) + 3.0
x = orc.cell_centers(dims, sp, org).T
y = x[None] + 0.4 * rng.standard_normal((K,) + x.shape) * np.asarray(sp)[None, :, None]
w = rng.uniform(0.5, 1.0, K)
fd = srb.DeviceFrames.from_array(srb.get_engine(), frames, srb.GridSpec(dims, sp, org), torch.float32)
obj = srb.FieldObjective(fd, list(range(K)), w, float(np.prod(sp)))
yt = torch.as_tensor(y).to(device=fd.data.device, dtype=torch.float32).contiguous()
stats, g = obj.evaluate(yt)
torch.cuda.synchronize()
q = frames.astype(np.float32).astype(np.float64)
_, Dref, gref = orc.evaluate_field(list(q), dims, sp, org, y.astype(np.float32).astype(np.float64), w, float(np.prod(sp)))
gd = g.double().cpu().numpy()
print("dD", abs(float(stats[0]) - Dref) / abs(Dref), "dg", float(np.abs(gd - gref).max() / np.abs(gref).max()))
