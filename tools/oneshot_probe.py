"""Wall time of the one-shot spmv_csrc (plan-free streamed path) at a config,
first and repeated calls, vs the plan-based paths."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1003_0952_b200 as P
from oracle.oracle import Oracle, rel_l2
cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
a, x, _ = P.config_matrix(cfg)
ref = Oracle().spmv_csrc(a, x)
for i in range(4):
    t0 = time.perf_counter(); y = P.spmv_csrc(a, x); dt = time.perf_counter() - t0
    print(f"oneshot call {i}: {dt*1e3:8.1f} ms  err {rel_l2(y, ref):.2e}", flush=True)
t0 = time.perf_counter(); yt = P.spmv_csrc_transpose(a, x); print(f"oneshot transpose: {(time.perf_counter()-t0)*1e3:8.1f} ms", flush=True)
for kind in ("gather", "windowed", "atomic"):
    t0 = time.perf_counter(); ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind[kind])); tp = time.perf_counter() - t0
    t0 = time.perf_counter(); y = ex.apply(x); ta = time.perf_counter() - t0
    print(f"plan {kind:8s}: create {tp*1e3:8.1f} ms + first apply {ta*1e3:8.1f} ms  err {rel_l2(y, ref):.2e}", flush=True)
    ex.close()
