"""Plan-build phase times (CSRC_GPU_PLAN_TRACE=1) for the gather plan."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CSRC_GPU_PLAN_TRACE"] = "1"
import paper_1003_0952_b200 as P
for cfg in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c5"]):
    a, x, _ = P.config_matrix(cfg)
    for kind in ("gather", "windowed"):
        t = time.time()
        ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind[kind]))
        print(f"{cfg} {kind} plan total {time.time() - t:.2f} s", flush=True)
        ex.close()
