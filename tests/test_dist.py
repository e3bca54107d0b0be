"""Multi-rank path on CPU (gloo, world size 2 and 3): the halo plan and the
P2P exchange of paper_1003_0952_b200.dist reassemble the full product; the
band product itself is injected from the oracle here (on the GPU box the band
plans of the windowed kernel do it; tests/test_gpu_parity.py checks those)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1003_0952_b200 as P
from paper_1003_0952_b200.dist import halo_plan

from .helpers import meshes


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _band_product(a, plan, x_local):
    """Oracle product of rows [row_begin, row_end) only, on [lo, row_end)."""
    from oracle.oracle import Oracle
    ia = a.ia.copy()
    ia[: plan.row_begin + 1] = a.ia[plan.row_begin]
    ia[plan.row_end + 1:] = a.ia[plan.row_end]
    ia = ia - ia[0]
    t0, t1 = a.ia[plan.row_begin], a.ia[plan.row_end]
    ad = np.zeros(a.n)
    ad[plan.row_begin:plan.row_end] = a.ad[plan.row_begin:plan.row_end]
    sub = P.CsrcMatrix(a.n, ad, ia, a.ja[t0:t1], a.al[t0:t1], a.au[t0:t1])
    x = np.zeros(a.n)
    x[plan.lo:plan.row_end] = x_local
    return Oracle().spmv_csrc(sub, x)[plan.lo:plan.row_end]


def _worker(rank, world, port, mesh_key, out_q):
    import torch
    import torch.distributed as dist
    from paper_1003_0952_b200.dist import DistSpmv

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = meshes()
        a = m.matrix(mesh_key)
        x = m[mesh_key + "x"]
        ds = DistSpmv(a, band_compute=lambda plan, xl: _band_product(a, plan, xl))
        p = ds.plan
        xl = torch.from_numpy(x[p.lo:p.row_end].copy())
        yl = torch.zeros_like(xl)
        ds.apply_host(xl, yl)
        out_q.put((rank, p.row_begin, p.row_end, yl.numpy()[p.row_begin - p.lo:].copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mesh_key", ["g1_", "g3_", "g5_"])
def test_gloo_band_exchange_reassembles_the_product(world, mesh_key):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mesh_key, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    parts = [q.get(timeout=120) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    m = meshes()
    y = np.zeros(int(m[mesh_key + "y"].size))
    for _, r0, r1, own in parts:
        y[r0:r1] = own
    ref = m[mesh_key + "y"]
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)


def test_halo_plan_is_consistent_across_ranks():
    m = meshes()
    a = m.matrix("g5_")
    for world in (2, 4, 8):
        plans = [halo_plan(a, world, r) for r in range(world)]
        sends = sorted((r, peer, q0, q1) for r, p in enumerate(plans) for peer, q0, q1 in p.sends)
        recvs = sorted((peer, r, q0, q1) for r, p in enumerate(plans) for peer, q0, q1 in p.recvs)
        assert sends == recvs  # every send has the matching receive
        assert plans[0].row_begin == 0 and plans[-1].row_end == a.n
        for p in plans:
            for peer, q0, q1 in p.sends:
                assert peer < p.rank and plans[peer].row_begin <= q0 < q1 <= plans[peer].row_end
