"""Host API with pageable vs pinned host vectors (the reference's API passes
std::vector, i.e. pageable memory)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1003_0952_b200 as P  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
a, x, _ = P.config_matrix(cfg)
ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind.gather))
xp = np.array(x)
yp = np.empty_like(xp)
xh = torch.from_numpy(x.copy()).pin_memory()
yh = torch.empty_like(xh).pin_memory()


def med(fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return sorted(ts)[len(ts) // 2] * 1e3


print(f"{cfg} pinned   x/y: {med(lambda: ex.apply(xh.numpy(), yh.numpy())):7.3f} ms", flush=True)
print(f"{cfg} pageable x/y: {med(lambda: ex.apply(xp, yp)):7.3f} ms", flush=True)
print(f"{cfg} pageable, fresh y each call: {med(lambda: ex.apply(xp)):7.3f} ms", flush=True)
