"""Host-API (e2e) pipeline variants for the gather plan: copy streams per
direction and chunk schedules (CSRC_GPU_HOST_*), wall time per product with
pinned x / y. Diagnostics for DESIGN.md §5 host path."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1003_0952_b200 as P  # noqa: E402


def timeit(fn, reps=30):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    ts.sort()
    return ts[len(ts) // 2]


cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
a, x, _ = P.config_matrix(cfg)
xh = torch.from_numpy(x).pin_memory()
yh = torch.empty_like(xh).pin_memory()
schedules = ["", "1,2,4,8,8,8,8,8,8,4,2,2,1,1", "1,1,2,4,8,8,8,8,8,8,4,2,1,1,1", "2,4,8,16,16,8,4,2,2,1,1",
             "1,2,3,4,4,4,4,4,4,4,4,4,4,4,4,3,2,1,1", "4,8,8,8,8,8,8,8,4,2,2,1,1"]
if len(sys.argv) > 2:  # schedules given as ';'-separated unit lists ('' = the default)
    schedules = sys.argv[2].split(";")
streams = ((1, 1), (2, 1), (1, 2), (2, 2)) if len(sys.argv) <= 3 else ((1, 1),)
for sch in schedules:
    if sch:
        os.environ["CSRC_GPU_HOST_UNITS"] = sch
    else:
        os.environ.pop("CSRC_GPU_HOST_UNITS", None)
    ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind.gather))
    for h2, d2 in streams:
        os.environ["CSRC_GPU_HOST_H2D_STREAMS"] = str(h2)
        os.environ["CSRC_GPU_HOST_D2H_STREAMS"] = str(d2)
        t = timeit(lambda: ex.apply(xh.numpy(), yh.numpy()))
        print(f"{cfg} units [{sch or 'default'}] h2d_streams {h2} d2h_streams {d2}: {t * 1e3:7.3f} ms", flush=True)
    ex.close()
