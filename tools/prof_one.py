"""Run one strategy on one config a few times (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1003_0952_b200 as P
cfg, kind = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dtype = P.DType.f32 if (len(sys.argv) > 4 and sys.argv[4] == 'f32') else P.DType.f64
a, x, _ = P.config_matrix(cfg)
ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind[kind], p=8, dtype=dtype))
xd = torch.from_numpy(x).cuda()
if dtype == P.DType.f32: xd = xd.float()
yd = torch.zeros_like(xd)
for _ in range(reps):
    ex.apply_device(xd, yd)
torch.cuda.synchronize()
print('ok', cfg, kind, ex.info().bands)
