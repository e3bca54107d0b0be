"""Multi-rank path on CPU (gloo, world size 2 and 3): the band forms of
paper_1003_0952_b200.dist reassemble the full product — the windowed form
through its halo plan and P2P exchange, the gather form with no exchange (x
replicated over [lo, x_hi)). The band product itself is injected from the
oracle here (on the GPU box the band plans do it; tests/test_gpu_parity.py
checks those)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1003_0952_b200 as P
from paper_1003_0952_b200.dist import band_x_hi, gather_plan, halo_plan

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


def _gather_band_product(a, plan, x_local):
    """Oracle product of rows [row_begin, row_end) from x on [lo, x_hi)."""
    from oracle.oracle import Oracle
    x = np.zeros(a.n)
    x[plan.x_lo:plan.x_hi] = x_local
    return Oracle().spmv_csrc(a, x)[plan.row_begin:plan.row_end]


def _worker(rank, world, port, mesh_key, out_q, mode="windowed", refresh=False):
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
        fn = _gather_band_product if mode == "gather" else _band_product
        s = P.Strategy(P.StrategyKind.gather if mode == "gather" else P.StrategyKind.windowed)
        ds = DistSpmv(a, s, band_compute=lambda plan, xl: fn(a, plan, xl))
        p = ds.plan
        assert p.mode == mode
        xl = torch.from_numpy(x[p.x_lo:p.x_hi].copy())
        if refresh:  # only the owned x rows are current; the halo comes from the peers
            xl[:] = float("nan")
            xl[p.row_begin - p.x_lo:p.row_end - p.x_lo] = torch.from_numpy(x[p.row_begin:p.row_end])
        yl = torch.zeros(p.row_end - p.y_lo, dtype=torch.float64)
        ds.apply_host(xl, yl, refresh_x=refresh)
        if refresh:
            assert np.array_equal(xl.numpy(), x[p.x_lo:p.x_hi])
        out_q.put((rank, p.row_begin, p.row_end, yl.numpy()[p.row_begin - p.y_lo:].copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["windowed", "gather", "gather_refresh"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mesh_key", ["g1_", "g3_", "g5_"])
def test_gloo_band_exchange_reassembles_the_product(world, mesh_key, mode):
    """gather_refresh: each rank starts with x current only on its own rows and
    the x halo arrives through the grouped P2P exchange (iterative use)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    refresh = mode == "gather_refresh"
    mode = "gather" if refresh else mode
    procs = [ctx.Process(target=_worker, args=(r, world, port, mesh_key, q, mode, refresh)) for r in range(world)]
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


def test_gather_plan_ranges():
    """Gather bands: no exchange; x range covers every column the band's rows
    read (lower pairs down to lo, upper pairs up to x_hi - 1)."""
    m = meshes()
    a = m.matrix("g3_")
    rows = np.repeat(np.arange(a.n), np.diff(a.ia))
    for world in (2, 3, 5):
        for r in range(world):
            p = gather_plan(a, world, r)
            assert not p.sends and not p.recvs and p.y_lo == p.row_begin
            lower = a.ja[a.ia[p.row_begin]:a.ia[p.row_end]]
            assert lower.size == 0 or lower.min() >= p.x_lo
            upper_rows = rows[(a.ja >= p.row_begin) & (a.ja < p.row_end)]
            assert upper_rows.size == 0 or upper_rows.max() < p.x_hi
            assert p.x_hi == band_x_hi(a, p.row_begin, p.row_end) >= p.row_end


def test_gather_x_halo_lists_are_consistent():
    """Every x row a rank receives is sent by its owner, exactly once, and the
    received pieces tile the rank's x range minus its own rows."""
    m = meshes()
    a = m.matrix("g5_")
    for world in (2, 3, 5, 8):
        plans = [gather_plan(a, world, r) for r in range(world)]
        sends = sorted((r, peer, q0, q1) for r, p in enumerate(plans) for peer, q0, q1 in p.x_sends)
        recvs = sorted((peer, r, q0, q1) for r, p in enumerate(plans) for peer, q0, q1 in p.x_recvs)
        assert sends == recvs
        for p in plans:
            covered = np.zeros(a.n, np.int32)
            covered[p.row_begin:p.row_end] += 1
            for peer, q0, q1 in p.x_recvs:
                assert plans[peer].row_begin <= q0 < q1 <= plans[peer].row_end
                covered[q0:q1] += 1
            assert np.all(covered[p.x_lo:p.x_hi] == 1)
            assert covered[:p.x_lo].sum() == 0 and covered[p.x_hi:].sum() == 0


def test_bands_x_hi_matches_the_numpy_definition():
    """csrc_bands_x_hi (threaded C++) equals the per-band numpy definition."""
    from paper_1003_0952_b200.dist import band_x_hi, bands_x_hi
    for cfg in ("c1", "c2"):
        a, _, _ = P.config_matrix(cfg)
        for p in (1, 2, 3, 8, 16):
            bs = P.partition_by_nnz(a, p).block_start
            assert bands_x_hi(a, bs) == [band_x_hi(a, bs[b], bs[b + 1]) for b in range(p)]


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_c_abi_exchange_lists_match_the_python_plans(cfg):
    """The C-ABI band executor (csrc/bandexec.cpp) derives the same exchange
    lists as paper_1003_0952_b200.dist (halo_plan / gather_plan)."""
    from paper_1003_0952_b200.dist import band_lists, gather_plan, halo_plan
    a, _, _ = P.config_matrix(cfg)
    for world in (1, 2, 3, 5, 8):
        for rank in range(world):
            info, sends, recvs = band_lists(a, world, rank, "windowed")
            h = halo_plan(a, world, rank)
            assert (sends, recvs) == (h.sends, h.recvs)
            assert (info.row_begin, info.row_end, info.lo, info.y_lo) == (h.row_begin, h.row_end, h.lo, h.lo)
            info, sends, recvs = band_lists(a, world, rank, "gather")
            g = gather_plan(a, world, rank)
            assert sorted(sends) == sorted(g.x_sends) and sorted(recvs) == sorted(g.x_recvs)
            assert (info.x_lo, info.x_hi, info.y_lo) == (g.x_lo, g.x_hi, g.y_lo)
