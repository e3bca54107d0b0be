"""Does a bandwidth-bound kernel slow the host-link copies? Times 128 MiB
copies each way (alone, both at once) with and without the C5 gather product
running back to back on a third stream, then the host-API product under
CSRC_GPU_HOST_GRID_DIV (chunk products on a fraction of the grid)."""
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
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
a, x, _ = P.config_matrix("c5")
ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind.gather))
xd = torch.from_numpy(x).cuda()
yd = torch.empty_like(xd)


def copies(which, with_kernel):
    torch.cuda.synchronize()
    if with_kernel:
        for _ in range(12):  # ~8 ms of products, longer than the copies
            ex.apply_device(xd, yd, s3)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    if "h" in which:
        e[0].record(s1)
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        e[1].record(s1)
    if "d" in which:
        e[2].record(s2)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        e[3].record(s2)
    torch.cuda.synchronize()
    out = []
    if "h" in which:
        out.append(nbytes / (e[0].elapsed_time(e[1]) / 1e3) / 1e9)
    if "d" in which:
        out.append(nbytes / (e[2].elapsed_time(e[3]) / 1e3) / 1e9)
    return out


for which in ("h", "d", "hd"):
    for k in (False, True):
        r = [copies(which, k) for _ in range(5)][1:]
        med = np.median(np.array(r), axis=0)
        print(f"copies {which:2s} kernel={'on ' if k else 'off'}: " + "  ".join(f"{v:6.1f} GB/s" for v in med),
              flush=True)

xh = torch.from_numpy(x).pin_memory()
yh = torch.empty_like(xh).pin_memory()
ex.close()
for div in (1, 2, 4, 8, 16):
    os.environ["CSRC_GPU_HOST_GRID_DIV"] = str(div)
    e2 = P.GpuSpmv(a, P.Strategy(P.StrategyKind.gather))
    e2.apply(xh.numpy(), yh.numpy())
    ts = []
    for _ in range(30):
        t = time.perf_counter()
        e2.apply(xh.numpy(), yh.numpy())
        ts.append(time.perf_counter() - t)
    print(f"host apply grid/{div:2d}: median {1e3*np.median(ts):7.3f} ms  min {1e3*min(ts):7.3f} ms", flush=True)
    if div in (1, 4):
        os.environ["CSRC_GPU_HOST_TRACE"] = "1"
        e2.apply(xh.numpy(), yh.numpy())
        del os.environ["CSRC_GPU_HOST_TRACE"]
    e2.close()
