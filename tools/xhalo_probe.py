"""Host-API product with halo-aligned x chunks (CSRC_GPU_HOST_XHALO=1, default)
vs row-aligned x chunks (0), C5 and C3, pinned and pageable vectors, fp64 and
fp32; median wall ms of 30 products, plus one traced call per variant at C5."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1003_0952_b200 as P

for cfg in ("c5", "c3"):
    a, x, _ = P.config_matrix(cfg)
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    for dt in (P.DType.f64, P.DType.f32):
        for rnd in range(2):
            for xhalo in ("0", "1"):
                os.environ["CSRC_GPU_HOST_XHALO"] = xhalo
                ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind.gather, dtype=dt))
                for pinned in (True, False):
                    xv, yv = (xh.numpy(), yh.numpy()) if pinned else (x.copy(), np.empty_like(x))
                    ex.apply(xv, yv)
                    ts = []
                    for _ in range(30):
                        t = time.perf_counter()
                        ex.apply(xv, yv)
                        ts.append(time.perf_counter() - t)
                    print(f"{cfg} {dt.name} xhalo={xhalo} {'pinned  ' if pinned else 'pageable'} round {rnd}: "
                          f"median {1e3*np.median(ts):7.3f} ms  min {1e3*min(ts):7.3f} ms", flush=True)
                if cfg == "c5" and dt == P.DType.f64 and rnd == 0:
                    os.environ["CSRC_GPU_HOST_TRACE"] = "1"
                    ex.apply(xh.numpy(), yh.numpy())
                    del os.environ["CSRC_GPU_HOST_TRACE"]
                ex.close()
