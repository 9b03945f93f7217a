"""Diagnostic (GPU box): cProfile of one warm C5 multilevel run (where the host time outside the solves goes)."""
import cProfile, pstats, sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2001_06613_b200 as srb
from paper_2001_06613_b200 import synth, multilevel as ml
from paper_2001_06613_b200.optimizer import OptimOptions
cfg = synth.CONFIGS['c5']
dev = torch.device('cuda', 0)
frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device=dev)
host = frames.to(cfg.dtype).cpu().pin_memory()
fcfg = ml.FieldRunConfig(spatial_levels=4, temporal_coarsest_size=9, feature=cfg.feature, ngf_eps=cfg.ngf_eps,
                         alpha=cfg.alpha, weights="uniform", eps=None,
                         optim=OptimOptions(max_iters=10, grad_tol=1e-30, f_tol=1e-30, step_tol=1e-30))
eng = srb.get_engine(0)
grid = srb.GridSpec(cfg.dims, spacing, origin)
def one_run():
    fd = srb.DeviceFrames(eng, host.to(dev, non_blocking=True), grid)
    y, runs = ml.field_stml_run(fd, times, fcfg)
    return y.cpu(), runs
for _ in range(2): one_run()
torch.cuda.synchronize()
t0 = time.perf_counter(); pr = cProfile.Profile(); pr.enable(); one_run(); pr.disable(); print('run s', time.perf_counter() - t0)
pstats.Stats(pr).sort_stats('cumulative').print_stats(28)
