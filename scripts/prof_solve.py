"""Diagnostic (GPU box): the pieces of one regularised objective call of the C5 finest level (y = c x, sr_evaluate_reg,
value readback, gradient scaling), two solver vector operations, and the per-kernel device times of the evaluation."""
import sys, time, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2001_06613_b200 as srb
from paper_2001_06613_b200 import synth, multilevel as ml
from paper_2001_06613_b200.field import FieldObjective
cfg = synth.CONFIGS['c5']
dev = torch.device('cuda', 0)
frames, times, spacing, origin = synth.make_sequence(cfg, seed=0, device=dev)
eng = srb.get_engine(0)
grid = srb.GridSpec(cfg.dims, spacing, origin)
fd = srb.DeviceFrames(eng, frames.to(cfg.dtype), grid)
K = cfg.K
w = np.full(K, 1.0 / K)
obj = FieldObjective(fd, list(range(K)), w, feature='ngf', ngf_eps=cfg.ngf_eps, alpha=10.0)
shape = obj.shape
n = int(np.prod(shape))
x = ml._identity(grid, K, torch.float64, dev, 0.3).reshape(-1).contiguous()
y = torch.empty(shape, dtype=torch.float32, device=dev)
g = torch.empty(shape, dtype=torch.float32, device=dev)
gout = torch.empty(n, dtype=torch.float64, device=dev)
c = 0.37
def sync(): torch.cuda.synchronize()
for rep in range(3):
    sync(); t0 = time.perf_counter()
    torch.mul(x.view(shape), c, out=y); sync(); t1 = time.perf_counter()
    stats, _ = obj.evaluate(y, g); sync(); t2 = time.perf_counter()
    v = float((stats[0] + obj.s_reg[0]).item()); t3 = time.perf_counter()
    torch.mul(g.reshape(-1), c, out=gout); sync(); t4 = time.perf_counter()
    print('mul y %.2f  evaluate %.2f  item %.2f  mul g %.2f ms' % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3, (t4-t3)*1e3))
# solver vector ops: x + t p
p = torch.randn(n, dtype=torch.float64, device=dev); xn = torch.empty_like(x)
sync(); t0 = time.perf_counter(); torch.add(x, p, alpha=0.5, out=xn); sync(); print('step %.2f ms' % ((time.perf_counter()-t0)*1e3))
sync(); t0 = time.perf_counter(); d = torch.dot(x, p).item(); print('dot %.2f ms' % ((time.perf_counter()-t0)*1e3))
from torch.profiler import ProfilerActivity, profile
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        obj.evaluate(y, g)
    torch.cuda.synchronize()
agg = {}
for ev in prof.events():
    if ev.device_type.name == "CUDA":
        agg.setdefault(ev.name[:60], []).append(ev.device_time * 1e-3)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print('%-62s n=%d  mean %.3f ms' % (k, len(v), sum(v) / len(v)))
