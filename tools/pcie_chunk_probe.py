"""Host-link copies in chunks: does splitting 128 MiB each way into the host
pipeline's chunk schedule (or N equal chunks) cost bandwidth when both
directions run at once? No kernels, no dependencies between the directions."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

n = 16 << 20  # doubles = 128 MiB
h1 = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d1 = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()


def bounds(units):
    tot = sum(units)
    b, acc = [0], 0
    for u in units:
        acc += u
        b.append(n * acc // tot)
    return b


def run(units_h, units_d, events=False, reps=10):
    bh, bd = bounds(units_h), bounds(units_d)
    ev = [torch.cuda.Event() for _ in range(64)]
    ts = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        t = time.perf_counter()
        with torch.cuda.stream(sa):
            for i in range(len(bh) - 1):
                d1[bh[i]:bh[i + 1]].copy_(h1[bh[i]:bh[i + 1]], non_blocking=True)
                if events:
                    ev[i].record(sa)
        with torch.cuda.stream(sb):
            for i in range(len(bd) - 1):
                h2[bd[i]:bd[i + 1]].copy_(d2[bd[i]:bd[i + 1]], non_blocking=True)
        torch.cuda.synchronize()
        if r:
            ts.append(time.perf_counter() - t)
    return 1e3 * float(np.median(ts))


sched = [2, 4, 8, 8, 8, 8, 8, 8, 4, 2, 2, 1, 1]

for name, uh, ud, ev in (("1 + 1", [1], [1], False),
                         ("pipeline schedule both", sched, sched, False),
                         ("pipeline schedule + events", sched, sched, True),
                         ("8 equal both", [1] * 8, [1] * 8, False),
                         ("32 equal both", [1] * 32, [1] * 32, False),
                         ("h2d sched, d2h 1", sched, [1], False),
                         ("h2d 1, d2h sched", [1], sched, False)):
    print(f"{name:28s}: {run(uh, ud, ev):7.3f} ms", flush=True)
