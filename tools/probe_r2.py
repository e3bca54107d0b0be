"""GPU probe (round 2): parity vs the oracle + sustained / cold timings for
kernel kinds under environment variants.

  python tools/probe_r2.py c2,c5 'colorful' 'wave:;old:CSRC_GPU_COLOR_WAVE=0;s32:CSRC_GPU_CW_S=32'
kinds: gather windowed atomic colorful colorful_exact lb_all_in_one lb_per_buffer lb_effective lb_interval
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1003_0952_b200 as P  # noqa: E402
from oracle.oracle import Oracle, rel_l2  # noqa: E402

O = Oracle()
K, A = P.StrategyKind, P.AccumMethod
KINDS = {
    "gather": P.Strategy(K.gather), "windowed": P.Strategy(K.windowed), "atomic": P.Strategy(K.atomic),
    "colorful": P.Strategy(K.colorful, p=8),
    "colorful_exact": P.Strategy(K.colorful, p=8, conflict_mode=P.ConflictMode.exact),
    "lb_all_in_one": P.Strategy(K.local_buffers, A.all_in_one, p=8),
    "lb_per_buffer": P.Strategy(K.local_buffers, A.per_buffer, p=8),
    "lb_effective": P.Strategy(K.local_buffers, A.effective, p=8),
    "lb_interval": P.Strategy(K.local_buffers, A.interval, p=8),
}
cfgs = sys.argv[1].split(",")
kinds = sys.argv[2].split(",")
variants = [v.split(":", 1) for v in (sys.argv[3] if len(sys.argv) > 3 else "default:").split(";")]
dtype = P.DType.f32 if os.environ.get("DT") == "f32" else P.DType.f64
reps = int(os.environ.get("REPS", "50"))
for cfg in cfgs:
    a, x, _ = P.config_matrix(cfg)
    if dtype == P.DType.f32:
        x = x.astype(np.float32).astype(np.float64)
        a32 = P.CsrcMatrix(a.n, a.ad.astype(np.float32).astype(np.float64), a.ia, a.ja,
                           a.al.astype(np.float32).astype(np.float64), a.au.astype(np.float32).astype(np.float64))
        ref = O.spmv_csrc(a32, x)
    else:
        ref = O.spmv_csrc(a, x)
    mb = P.model_bytes(a, dtype)
    tdt = torch.float32 if dtype == P.DType.f32 else torch.float64
    xd = torch.from_numpy(x).to("cuda", tdt)
    yd = torch.zeros_like(xd)
    flush = 0 if mb > 400e6 else 256 << 20
    print(f"== {cfg} n={a.n} model {mb / 1e6:.1f} MB flush {flush >> 20} MB", flush=True)
    for kn in kinds:
        for vname, venv in variants:
            env = dict(kv.split("=", 1) for kv in venv.split(",") if kv)
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                s = KINDS[kn]
                s = P.Strategy(s.kind, s.accum, p=s.p, dtype=dtype, conflict_mode=s.conflict_mode)
                t0 = time.time()
                ex = P.GpuSpmv(a, s)
                tp = time.time() - t0
                y = ex.apply(x)
                err = rel_l2(y, ref)
                y2 = ex.apply(x)
                bitrep = bool(np.array_equal(y, y2))
                for _ in range(3):
                    ex.apply_device(xd, yd)
                tot, ker = ex.time_products(xd, yd, reps, flush)
                inf = ex.info()
                ms, kms = float(np.mean(tot[2:])), float(np.mean(ker[2:]))
                mn = float(np.min(ker[2:]))
                print(f"  {kn:15s} {vname:10s} err {err:.2e} rep {int(bitrep)} plan {tp:6.2f}s "
                      f"step {ms * 1e3:8.1f}us kernel {kms * 1e3:8.1f}us (min {mn * 1e3:8.1f}) "
                      f"{mb / kms / 1e6:7.1f} GB/s frac {mb / kms / 1e6 / 6551.7:.3f} colors {inf.n_colors} "
                      f"bands {inf.bands} dev {inf.device_bytes / 1e9:.2f} GB", flush=True)
                ex.close()
            except Exception as e:  # noqa: BLE001
                print(f"  {kn:15s} {vname:10s} FAILED: {e}", flush=True)
            finally:
                for k, v in old.items():
                    if v is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = v
