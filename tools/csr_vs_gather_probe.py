"""C5: CSRC gather plan vs CSR plan of the same matrix (diagonal in the entry
stream), sustained kernel times over 300 products each, interleaved twice."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1003_0952_b200 as P  # noqa: E402
from oracle.oracle import Ref  # noqa: E402

a, x, _ = P.config_matrix(sys.argv[1] if len(sys.argv) > 1 else "c5")
n, _, r, c, v = P.csrc_to_triplets(a)
m = P.build_csr((n, n, r, c, v))
del r, c, v
xd = torch.from_numpy(x).cuda()
yd = torch.zeros_like(xd)
plans = {"csrc-gather": P.GpuSpmv(a, P.Strategy(P.StrategyKind.gather)),
         "csr": P.GpuSpmv(m, P.Strategy(P.StrategyKind.gather))}
for rnd in range(2):
    for name, ex in plans.items():
        for _ in range(10):
            ex.apply_device(xd, yd)
        tot, ker = ex.time_products(xd, yd, 300, 0)
        k = ker * 1e3
        print(f"round {rnd} {name:12s} mean {k.mean():6.1f} median {np.median(k):6.1f} first50 {k[:50].mean():6.1f} "
              f"last250 {k[50:].mean():6.1f} us  patterns {ex.info().row_patterns}", flush=True)
