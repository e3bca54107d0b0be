"""Host link bandwidth (pinned H2D, D2H, both directions at once) and the
gather plan's host-API product time, for the e2e analysis in DESIGN.md."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1003_0952_b200 as P

nbytes = 128 << 20
h1 = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
h2 = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
d1 = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
d2 = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=20):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)


def both():
    h2d(); d2h()


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    t = timeit(fn)
    print(f"{name:5s} 128 MiB each: {t*1e3:7.3f} ms  {nbytes/t/1e9:6.1f} GB/s per direction")

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
a, x, _ = P.config_matrix(cfg)
xh = torch.from_numpy(x).pin_memory()
yh = torch.empty_like(xh).pin_memory()
for chunks in (1, 8, 16, 0):  # 0 = default ramped schedule
    os.environ["CSRC_GPU_HOST_CHUNKS"] = str(chunks)
    ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind.gather))
    t = timeit(lambda: ex.apply(xh.numpy(), yh.numpy()), reps=20)
    print(f"{cfg} host apply, chunks<={chunks:2d}: {t*1e3:7.3f} ms")
    ex.close()

os.environ["CSRC_GPU_HOST_CHUNKS"] = "0"
ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind.gather))
ex.apply(xh.numpy(), yh.numpy())
os.environ["CSRC_GPU_HOST_TRACE"] = "1"
ex.apply(xh.numpy(), yh.numpy())
t = time.perf_counter(); ex.apply(xh.numpy(), yh.numpy()); print(f"traced call wall {1e3*(time.perf_counter()-t):.3f} ms", flush=True)
del os.environ["CSRC_GPU_HOST_TRACE"]
t = time.perf_counter(); ex.apply(xh.numpy(), yh.numpy()); print(f"untraced call wall {1e3*(time.perf_counter()-t):.3f} ms", flush=True)
