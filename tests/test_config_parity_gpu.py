"""Full-size parity of the default CUDA path on the BASELINE configs C2, C3 and C4 (north_star: D, grad D
within 1e-4 relative in fp32 mode on the seeded synthetic sequences).

The fixture tests/golden/config_golden.npz is the CPU oracle (fp64 arithmetic on the same float32
inputs) run by tests/golden/make_config_golden.py; the inputs are regenerated here from the seeded
generator (synth.make_sequence, synth.bench_iterate: the iterate bench.py times) on the CPU, quantised
to float32 and uploaded.  The evaluation goes through the public device API (FieldObjective ->
sr_evaluate), i.e. exactly the kernels bench.py measures.  Pattern: /root/reference/pkg/tests/
test_similarity.py:113-130 (brute-force check of C), extended to D and the gradient.

Tolerances (written here): D relative 1e-4; C absolute 1e-4; gradient entries (sampled indices and the
stored slab) within 1e-4 of max |dD/dy|; per-frame gradient norms relative 1e-4.
"""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tests" / "golden"))

pytestmark = pytest.mark.gpu

GOLD = ROOT / "tests" / "golden" / "config_golden.npz"
TOL = 1e-4


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_config_full_size(name, gold):
    import make_config_golden as mk

    import paper_2001_06613_b200 as srb

    fr, yv, w, spacing, origin, cfg = mk.config_inputs(name)
    K, d, N = yv.shape
    dev = torch.device("cuda", 0)
    eng = srb.get_engine(0)
    fd = srb.DeviceFrames(eng, torch.as_tensor(fr, dtype=torch.float32).to(dev), srb.GridSpec(cfg.dims, spacing, origin))
    y = torch.as_tensor(yv, dtype=torch.float32).to(dev).contiguous()
    del fr, yv
    obj = srb.FieldObjective(fd, list(range(K)), w, float(np.prod(spacing)), feature=cfg.feature, ngf_eps=cfg.ngf_eps)
    for _ in range(3):  # eager, capture, replay: every path of sr_evaluate gives the same numbers
        stats, g = obj.evaluate(y)
        torch.cuda.synchronize()
        hs = obj.host_stats()
        D = hs["D"]
        Dref = float(gold[f"{name}/D"])
        assert abs(D - Dref) <= TOL * abs(Dref), (name, D, Dref)
        assert np.abs(hs["corr"] - gold[f"{name}/C"]).max() <= TOL
        gmax = float(gold[f"{name}/gmax"])
        gs = g.reshape(-1)[torch.as_tensor(mk.sample_index(K, d, N), device=dev)].double().cpu().numpy()
        err_s = np.abs(gs - gold[f"{name}/gsample"]).max() / gmax
        cells = torch.as_tensor(mk.slab_cells(cfg.dims), device=dev)
        slab = g[:, :, cells].double().cpu().numpy()
        err_slab = np.abs(slab - gold[f"{name}/gslab"]).max() / gmax
        gn = torch.linalg.vector_norm(g.double().reshape(K, -1), dim=1).cpu().numpy()
        err_n = np.abs(gn - gold[f"{name}/gnorm"]).max() / np.abs(gold[f"{name}/gnorm"]).max()
        assert err_s <= TOL and err_slab <= TOL and err_n <= TOL, (name, err_s, err_slab, err_n)
    print(f"{name}: D {D:.10g} vs {Dref:.10g}; grad err sample {err_s:.2e} slab {err_slab:.2e} norms {err_n:.2e}")
