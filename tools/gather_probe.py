"""Gather-kernel timing probe (env-driven variants): per config and dtype,
median kernel time over 50 products, model / layout GB/s. Diagnostics only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1003_0952_b200 as P  # noqa: E402

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c5"]
dts = sys.argv[2].split(",") if len(sys.argv) > 2 else ["f64"]
tag = os.environ.get("TAG", "")
for name in cfgs:
    a, x, _ = P.config_matrix(name)
    for dt in dts:
        dtype = P.DType.f32 if dt == "f32" else P.DType.f64
        tdt = torch.float32 if dt == "f32" else torch.float64
        ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind.gather, dtype=dtype))
        xd = torch.from_numpy(x).to(device="cuda", dtype=tdt)
        yd = torch.zeros_like(xd)
        for _ in range(5):
            ex.apply_device(xd, yd)
        mb = P.model_bytes(a, dtype)
        flush = 0 if mb > 400e6 else 256 << 20
        tot, ker = ex.time_products(xd, yd, 50, flush)
        k = float(np.median(ker[5:]))
        inf = ex.info()
        print(f"{tag:40s} {name} {dt} kernel {k * 1e3:8.1f} us  model {mb / k / 1e6:7.0f} GB/s  "
              f"layout {inf.stream_bytes / k / 1e6:7.0f} GB/s  L={inf.lanes} pat={inf.row_patterns}", flush=True)
        ex.close()
