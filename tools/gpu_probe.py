"""Quick GPU probe: parity of every kernel vs the oracle + event timings."""
import sys, time, json, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1003_0952_b200 as P
from oracle.oracle import Oracle, rel_l2
O = Oracle()
cfgs = sys.argv[1].split(',') if len(sys.argv) > 1 else ['c1', 'c2']
kinds = [('windowed', P.StrategyKind.windowed, 0), ('gather', P.StrategyKind.gather, 0), ('atomic', P.StrategyKind.atomic, 0),
         ('colorful', P.StrategyKind.colorful, 0), ('lb_effective', P.StrategyKind.local_buffers, 2),
         ('lb_interval', P.StrategyKind.local_buffers, 3), ('lb_all_in_one', P.StrategyKind.local_buffers, 0),
         ('lb_per_buffer', P.StrategyKind.local_buffers, 1)]
only = os.environ.get('KINDS')
if only: kinds = [k for k in kinds if k[0] in only.split(',')]
for name in cfgs:
    t = time.time(); a, x, _ = P.config_matrix(name); tg = time.time() - t
    t = time.time(); yref = O.spmv_csrc(a, x); to = time.time() - t
    mb = P.model_bytes(a)
    print(f'== {name} n={a.n} k={a.k_off()} gen {tg:.2f}s oracle {to:.2f}s model {mb/1e6:.1f} MB', flush=True)
    xd = torch.from_numpy(x).cuda(); yd = torch.zeros_like(xd)
    for kn, kind, acc in kinds:
        big = a.n > 5_000_000 and not os.environ.get('ALLBIG')
        if kind == P.StrategyKind.colorful and big: continue
        if kind == P.StrategyKind.local_buffers and big and acc in (0, 1): continue
        try:
            t = time.time(); ex = P.GpuSpmv(a, P.Strategy(kind, P.AccumMethod(acc), p=8)); tp = time.time() - t
            y = ex.apply(x)
            err = rel_l2(y, yref)
            ex.apply_device(xd, yd); torch.cuda.synchronize()
            err_d = rel_l2(yd.cpu().numpy(), yref)
            tot, ker = ex.time_products(xd, yd, 20, flush_bytes=0)
            totc, kerc = ex.time_products(xd, yd, 10, flush_bytes=256 << 20)
            inf = ex.info()
            hot = np.median(tot[3:]); cold = np.median(totc[2:]); kc = np.median(kerc[2:])
            print(f'  {kn:14s} err {err:.2e}/{err_d:.2e} plan {tp:.2f}s hot {hot*1e3:8.1f}us cold {cold*1e3:8.1f}us '
                  f'(kernel {kc*1e3:8.1f}us) cold GB/s {mb/cold/1e6:7.1f} warps {inf.bands} L {inf.lanes} st {inf.stages} '
                  f'smem {inf.smem_bytes} win {[(inf.win_lo[i], inf.win_hi[i]) for i in range(inf.n_windows)]} capt {inf.captured_fraction:.3f} colors {inf.n_colors}', flush=True)
            ex.close()
        except Exception as e:
            print(f'  {kn:14s} FAILED: {e}', flush=True)
    if os.environ.get('NOF32'): continue
    # fp32 windowed
    ex = P.GpuSpmv(a, P.Strategy(P.StrategyKind.windowed, dtype=P.DType.f32))
    x32 = x.astype(np.float32).astype(np.float64)
    a32 = P.CsrcMatrix(a.n, a.ad.astype(np.float32).astype(np.float64), a.ia, a.ja,
                       a.al.astype(np.float32).astype(np.float64), a.au.astype(np.float32).astype(np.float64))
    y = ex.apply(x32); print(f'  windowed f32   err {rel_l2(y, O.spmv_csrc(a32, x32)):.2e}', flush=True)
    xf = xd.float(); yf = torch.zeros_like(xf)
    totc, kerc = ex.time_products(xf, yf, 10, flush_bytes=256 << 20)
    mb32 = P.model_bytes(a, P.DType.f32)
    print(f'  windowed f32 cold {np.median(totc[2:])*1e3:.1f}us GB/s {mb32/np.median(totc[2:])/1e6:.1f}', flush=True)
    ex.close()
