"""Sustained-run drift of the C5 gather kernel for staged block sizes:
kernel-time percentiles and per-50-product means over 400 back-to-back
products (power / clock behaviour under load). Diagnostics."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1003_0952_b200 as P  # noqa: E402

a, x, _ = P.config_matrix("c5")
xd = torch.from_numpy(x).cuda()
yd = torch.zeros_like(xd)
# each argument: "KIND:ENV=V;ENV=V" (KIND gather|windowed), or a bare staged block size
for spec in sys.argv[1].split(","):
    kind, _, envs = spec.partition(":") if ":" in spec else ("gather", "", f"CSRC_GPU_GNT={spec}")
    saved = dict(os.environ)
    for kv in filter(None, envs.split(";")):
        k, v = kv.split("=")
        os.environ[k] = v
    ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind[kind]))
    os.environ.clear()
    os.environ.update(saved)
    nt = spec
    for _ in range(10):
        ex.apply_device(xd, yd)
    tot, ker = ex.time_products(xd, yd, 400, 0)
    k = ker * 1e3
    chunks = " ".join(f"{k[i:i + 50].mean():6.1f}" for i in range(0, 400, 50))
    print(f"GNT={nt:4s} mean {k.mean():6.1f} median {np.median(k):6.1f} p10 {np.percentile(k, 10):6.1f} "
          f"p90 {np.percentile(k, 90):6.1f} us | per-50 means: {chunks}", flush=True)
    ex.close()
