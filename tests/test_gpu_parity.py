"""GPU parity: every sm_100a kernel against the reference's own outputs
(golden vectors made by running the reference, tests/golden/) and against the
oracle. Tolerances (BASELINE.json north star): fp64 relative L2 <= 1e-12 (we
also require the reference's inf-norm 1e-12, bench.hpp:93-100); fp32 relative
L2 <= 1e-5 against the fp64 oracle on fp32-rounded inputs."""
import numpy as np
import pytest

from oracle.oracle import Oracle

import paper_1003_0952_b200 as P

from .helpers import family, known_answers, matrix_from_dict, meshes, rel_inf, rel_l2, round32

pytestmark = pytest.mark.gpu

O = Oracle()
KA = known_answers()
FAM = family()
MESH = meshes()
K = P.StrategyKind
A = P.AccumMethod

STRATEGIES = [
    ("sequential", P.Strategy(K.sequential)),
    ("windowed", P.Strategy(K.windowed)),
    ("gather", P.Strategy(K.gather)),
    ("atomic", P.Strategy(K.atomic)),
    ("colorful_nbh", P.Strategy(K.colorful, p=4)),
    ("colorful_exact", P.Strategy(K.colorful, p=4, conflict_mode=P.ConflictMode.exact)),
    ("lb_all_in_one", P.Strategy(K.local_buffers, A.all_in_one, p=4)),
    ("lb_per_buffer", P.Strategy(K.local_buffers, A.per_buffer, p=4)),
    ("lb_effective", P.Strategy(K.local_buffers, A.effective, p=4)),
    ("lb_interval", P.Strategy(K.local_buffers, A.interval, p=4)),
]
TOL64 = 1e-12
TOL32 = 1e-5


def run(a, x, s, transpose=False):
    ex = P.GpuSpmv(a, s)
    try:
        return ex.apply(x, transpose=transpose)
    finally:
        ex.close()


@pytest.mark.parametrize("name,s", STRATEGIES, ids=[n for n, _ in STRATEGIES])
def test_known_answers(name, s):
    for key in ("spmv_diag", "spmv_2x2"):
        ka = KA[key]
        a = matrix_from_dict(ka["matrix"])
        assert run(a, ka["x"], s).tolist() == ka["y"]


@pytest.mark.parametrize("name,s", STRATEGIES, ids=[n for n, _ in STRATEGIES])
@pytest.mark.parametrize("idx", range(29))
def test_family(name, s, idx):
    p = f"m{idx}_"
    a = FAM.matrix(p)
    for xk, yk in (("x", "y"), ("xr", "yr")):
        y = run(a, FAM[p + xk], s)
        assert rel_l2(y, FAM[p + yk]) <= TOL64
        assert rel_inf(y, FAM[p + yk]) <= TOL64


@pytest.mark.parametrize("idx", range(29))
def test_family_transpose(idx):
    p = f"m{idx}_"
    a = FAM.matrix(p)
    y = P.spmv_csrc_transpose(a, FAM[p + "xr"])
    assert rel_l2(y, FAM[p + "yt"]) <= TOL64
    for kind in (K.windowed, K.gather, K.atomic, K.colorful):
        y = run(a, FAM[p + "xr"], P.Strategy(kind, p=2), transpose=True)
        assert rel_l2(y, FAM[p + "yt"]) <= TOL64, kind.name


def test_gather_is_bit_reproducible():
    """The gather kernel has a fixed summation order per row: repeated
    products are bit-identical (no atomics anywhere)."""
    a = MESH.matrix("g5_")
    ex = P.GpuSpmv(a, P.Strategy(K.gather))
    y1 = ex.apply(MESH["g5_x"])
    for _ in range(5):
        assert np.array_equal(ex.apply(MESH["g5_x"]), y1)
    assert ex.info().launches_per_apply == 1
    ex.close()


@pytest.mark.parametrize("name,s", STRATEGIES, ids=[n for n, _ in STRATEGIES])
@pytest.mark.parametrize("idx", range(6))
def test_meshes(name, s, idx):
    p = f"g{idx}_"
    a = MESH.matrix(p)
    y = run(a, MESH[p + "x"], s)
    assert rel_l2(y, MESH[p + "y"]) <= TOL64


@pytest.mark.parametrize("kind", [K.windowed, K.gather, K.atomic, K.colorful])
@pytest.mark.parametrize("idx", range(6))
def test_meshes_fp32(kind, idx):
    p = f"g{idx}_"
    a = MESH.matrix(p)
    x32 = MESH[p + "x"].astype(np.float32).astype(np.float64)
    ref = O.spmv_csrc(round32(a), x32)
    y = run(a, x32, P.Strategy(kind, p=4, dtype=P.DType.f32))
    assert rel_l2(y, ref) <= TOL32


def test_p1_matches_the_reference_path():
    """p = 1 short-circuits (parallel.hpp:197-202): no buffers, same result."""
    a = MESH.matrix("g1_")
    ex = P.GpuSpmv(a, P.Strategy(K.local_buffers, A.effective, p=1))
    assert ex.buffers_allocated() == 0
    assert ex.info().launches_per_apply == 1  # runs the gather kernel
    assert rel_l2(ex.apply(MESH["g1_x"]), MESH["g1_y"]) <= TOL64
    ex.close()
    ex = P.GpuSpmv(a, P.Strategy(K.local_buffers, A.effective, p=4))
    assert ex.buffers_allocated() > 0
    ex.close()


def test_explicit_local_buffers_plan_2x2():
    """test_parallel.cpp:59-79: p=2, blocks {0},{1} -> (14, 5)."""
    ka = KA["spmv_2x2"]
    a = matrix_from_dict(ka["matrix"])
    part = P.RowPartition(2, [0, 1, 2], [1, 2])
    ranges = P.effective_ranges(a, part)
    plan = P.LocalBuffersPlan(part, ranges, P.build_interval_plan(ranges))
    for acc in A:
        ex = P.GpuSpmv(a, P.Strategy(K.local_buffers, acc, p=2), plan)
        assert ex.apply(ka["x"]).tolist() == [14.0, 5.0]
        assert ex.buffers_allocated() == 2
        ex.close()


@pytest.mark.parametrize("p", [2, 3, 8, 148, 1000])
def test_local_buffers_spill_form(p):
    """The GPU private buffers: the part of band b's buffer at or above its
    first row is y itself (no lower band writes there), the part below is a
    spill buffer of effective_range lo .. first row (partition.hpp:94-102).
    Every accumulation equals the oracle; the spill storage is the halo only,
    not p dense n-vectors."""
    a, x, _ = P.config_matrix("c2")
    ref = O.spmv_csrc(a, x)
    part = P.partition_by_nnz(a, p)
    rng = P.effective_ranges(a, part)
    halo = sum(max(0, part.begin(b) - r.lo) for b, r in enumerate(rng))
    for acc in A:
        ex = P.GpuSpmv(a, P.Strategy(K.local_buffers, acc, p=p))
        assert ex.buffers_allocated() == p
        y = ex.apply(x)
        assert rel_l2(y, ref) <= TOL64 and rel_inf(y, ref) <= TOL64, acc.name
        ex.close()
    # explicit uneven partition (LocalBuffersPlan given by the caller)
    cut = sorted(set([0, 1, 7, a.n // 3, a.n // 3 + 5, a.n - 2, a.n]))
    bs = P.RowPartition(len(cut) - 1, cut, [0] * (len(cut) - 1))
    r2 = P.effective_ranges(a, bs)
    plan = P.LocalBuffersPlan(bs, r2, P.build_interval_plan(r2))
    for acc in A:
        ex = P.GpuSpmv(a, P.Strategy(K.local_buffers, acc, p=bs.p), plan)
        assert rel_l2(ex.apply(x), ref) <= TOL64, acc.name
        ex.close()
    assert halo < p * 70_000  # C2 bandwidth 4161: the spill is the halo only


def test_mismatched_plans_throw():
    """test_parallel.cpp:159-165."""
    a = MESH.matrix("g0_")
    lb = P.LocalBuffersPlan.build(a, 3)
    with pytest.raises(P.Error, match="plan built for p=3, strategy has p=4"):
        P.GpuSpmv(a, P.Strategy(K.local_buffers, p=4), lb)
    with pytest.raises(P.Error, match="local-buffers plan given to a different strategy"):
        P.GpuSpmv(a, P.Strategy(K.colorful, p=3), lb)
    cp = P.ColorfulPlan.build(a, 3)
    with pytest.raises(P.Error, match="colorful plan given to a different strategy"):
        P.GpuSpmv(a, P.Strategy(K.local_buffers, p=3), cp)


@pytest.mark.parametrize("idx", range(29))
def test_explicit_colorings_all_orders(idx):
    p = f"m{idx}_"
    if not FAM.has(p + "col00"):
        pytest.skip("no colouring stored")
    a = FAM.matrix(p)
    for mode in (0, 1):
        for order in (0, 1, 2):
            plan = P.ColorfulPlan(P.Coloring(FAM[p + f"col{mode}{order}"], int(FAM[p + f"nc{mode}{order}"])))
            ex = P.GpuSpmv(a, P.Strategy(K.colorful, p=4), plan)
            assert ex.info().n_colors == plan.coloring.n_colors
            assert rel_l2(ex.apply(FAM[p + "x"]), FAM[p + "y"]) <= TOL64
            ex.close()


def test_corrupt_coloring_is_rejected():
    """bench_main.cpp:238-249 --corrupt-coloring: merged classes are detected."""
    a = MESH.matrix("g1_")
    c = P.color_rows(a)
    bad = c.color.copy()
    bad[bad == 1] = 0
    with pytest.raises(P.Error, match="coloring violation"):
        P.GpuSpmv(a, P.Strategy(K.colorful, p=2), P.ColorfulPlan(P.Coloring(bad, c.n_colors)))


def test_colorful_repeats_are_bit_identical():
    """test_parallel.cpp:115-123 (atomic-free variant)."""
    a = MESH.matrix("g5_")
    ex = P.GpuSpmv(a, P.Strategy(K.colorful, p=4))
    y1 = ex.apply(MESH["g5_x"])
    for _ in range(5):
        assert np.array_equal(ex.apply(MESH["g5_x"]), y1)
    ex.close()


def test_x_length_error():
    a = MESH.matrix("g0_")
    ex = P.GpuSpmv(a, P.Strategy(K.windowed))
    with pytest.raises(P.Error, match=f"x has length 3, expected {a.n}"):
        ex.apply(np.ones(3))
    ex.close()
    with pytest.raises(P.Error, match=f"spmv_csrc: x has length 3, expected {a.n}"):
        P.spmv_csrc(a, np.ones(3))


def test_timings_populated():
    """test_parallel.cpp:167-177."""
    a, x, _ = P.config_matrix("c2")
    for s in (P.Strategy(K.windowed), P.Strategy(K.local_buffers, A.interval, p=4)):
        ex = P.GpuSpmv(a, s)
        ex.set_timing(True)
        ex.apply(x)
        t = ex.last_timings()
        assert t.compute_max > 0 and t.init_max >= 0 and t.accumulate_max >= 0
        ex.close()


def test_edge_cases():
    # n = 0
    e = P.CsrcMatrix(0, [], [0], [], [], [])
    assert P.spmv_csrc(e, []).size == 0
    # n = 1, no pairs
    one = P.CsrcMatrix(1, [3.0], [0, 0], [], [], [])
    assert P.spmv_csrc(one, [2.0]).tolist() == [6.0]
    # rows without pairs in the middle, value-symmetric matrix
    a = P.CsrcMatrix(4, [1, 2, 3, 4], [0, 0, 1, 1, 3], [0, 0, 1], [0.5, 0.25, 0.125], [], True)
    x = np.array([1.0, -2.0, 3.0, 0.5])
    for name, s in STRATEGIES:
        assert rel_l2(run(a, x, s), O.spmv_csrc(a, x)) <= TOL64, name


@pytest.mark.parametrize("env", [{}, {"CSRC_GPU_GSELL": "1"}, {"CSRC_GPU_GSELL": "1", "CSRC_GPU_SELL_L": "2"},
                                 {"CSRC_GPU_GNT": "256"}])
def test_non_finite_x_and_ragged_sizes(env, monkeypatch):
    """inf / NaN in x propagate to exactly the rows the oracle marks (no
    padding or out-of-row slot is ever multiplied in), on sizes that are not
    multiples of a slice, a row block or a tile."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(11)
    for n in (1, 31, 33, 257, 1000):
        m = meshes().matrix("g1_")
        if n > m.n:
            continue
        # leading principal n x n block of a mesh matrix (rows keep their lower pairs < n)
        ia = m.ia[: n + 1].copy()
        k = int(ia[n])
        a = P.CsrcMatrix(n, m.ad[:n], ia, m.ja[:k], m.al[:k], m.au[:k])
        x = rng.uniform(-1, 1, n)
        x[n // 2] = np.inf
        if n > 2:
            x[n // 3] = np.nan
        ref = O.spmv_csrc(a, x)
        for kind in (K.gather, K.windowed, K.atomic, K.colorful):
            y = run(a, x, P.Strategy(kind, p=2 if kind == K.colorful else 1))
            assert np.array_equal(np.isnan(y), np.isnan(ref)), (n, kind)
            assert np.array_equal(np.isinf(y), np.isinf(ref)), (n, kind)
            fin = np.isfinite(ref)
            assert rel_l2(y[fin], ref[fin]) <= TOL64


@pytest.mark.parametrize("env", [{}, {"CSRC_GPU_GSELL": "1"}, {"CSRC_GPU_GNT": "256"}, {"CSRC_GPU_WIN_RINGS": "1"}])
def test_no_writes_outside_y(env, monkeypatch):
    """Out-of-bounds write check (compute-sanitizer is not available on the
    pool): y lives inside a larger buffer whose guard regions hold a sentinel;
    every kernel kind must leave them untouched, for sizes that are not
    multiples of a slice, row block or tile."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    guard = 4096
    for key in ("g1_", "g2_", "g4_"):
        a = MESH.matrix(key)
        x = torch.from_numpy(MESH[key + "x"]).cuda()
        for name, s in STRATEGIES:
            ex = P.GpuSpmv(a, s)
            buf = torch.full((a.n + 2 * guard,), 12345.0, dtype=torch.float64, device="cuda")
            ex.apply_device(x, buf[guard:guard + a.n])
            torch.cuda.synchronize()
            assert bool((buf[:guard] == 12345.0).all()) and bool((buf[guard + a.n:] == 12345.0).all()), (key, name)
            assert rel_l2(buf[guard:guard + a.n].cpu().numpy(), MESH[key + "y"]) <= TOL64, (key, name)
            ex.close()


@pytest.mark.parametrize("cfg", ["c2", "c3", "c4"])
def test_device_plan_build_equals_host_build(cfg, monkeypatch):
    """The opt-in device builder of whole-matrix gather plans
    (CSRC_GPU_PLAN_DEVICE=1: stable radix sort of the pairs by column) must
    give the host builder's plan: identical products, bit for bit, normal and
    transposed, fp64 and fp32."""
    import torch
    a, x, _ = P.config_matrix(cfg)
    xd = torch.from_numpy(x).cuda()
    for dt, tdt in ((P.DType.f64, torch.float64), (P.DType.f32, torch.float32)):
        out = []
        for dev_build in ("1", "0"):
            monkeypatch.setenv("CSRC_GPU_PLAN_DEVICE", dev_build)
            ex = P.GpuSpmv(a, P.Strategy(K.gather, dtype=dt))
            xin = xd.to(tdt)
            y = torch.empty_like(xin)
            yt = torch.empty_like(xin)
            ex.apply_device(xin, y)
            ex.apply_device(xin, yt, transpose=True)
            torch.cuda.synchronize()
            out.append((y.cpu().numpy(), yt.cpu().numpy(), ex.info().row_patterns, ex.info().gather_form))
            ex.close()
        assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1]), (cfg, dt)
        assert out[0][2:] == out[1][2:]
    assert rel_l2(out[0][0], O.spmv_csrc(round32(a), x.astype(np.float32).astype(np.float64))) <= TOL32


def test_device_and_graph_entry_points():
    import torch
    a, x, _ = P.config_matrix("c1")
    ref = O.spmv_csrc(a, x)
    for s in (P.Strategy(K.windowed), P.Strategy(K.gather), P.Strategy(K.atomic),
              P.Strategy(K.colorful, p=2), P.Strategy(K.local_buffers, A.effective, p=2)):
        ex = P.GpuSpmv(a, s)
        xd = torch.from_numpy(x).cuda()
        yd = torch.full_like(xd, float("nan"))
        st = torch.cuda.Stream()
        ex.apply_device(xd, yd, st)
        st.synchronize()
        assert rel_l2(yd.cpu().numpy(), ref) <= TOL64
        yd.fill_(float("nan"))
        for _ in range(3):
            ex.apply_device_graph(xd, yd, st)
        st.synchronize()
        assert rel_l2(yd.cpu().numpy(), ref) <= TOL64
        ex.close()


@pytest.mark.parametrize("kind", [K.windowed, K.gather, K.atomic, K.colorful, K.local_buffers])
@pytest.mark.parametrize("on_side_stream", [False, True])
def test_apply_device_is_ordered_on_torch_stream(kind, on_side_stream):
    """apply_device without a stream argument enqueues on torch's current
    stream (the default legacy NULL stream included), so torch ops queued
    after it see the product with no explicit synchronize in between."""
    import torch
    a, x, _ = P.config_matrix("c3")
    ref = O.spmv_csrc(a, x)
    ex = P.GpuSpmv(a, P.Strategy(kind, p=4))
    xd = torch.from_numpy(x).cuda()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side if on_side_stream else torch.cuda.current_stream()):
        outs = []
        for _ in range(3):
            y = torch.full_like(xd, float("nan"))
            ex.apply_device(xd * 1.0, y)  # x produced by a torch op on the same stream
            outs.append(y.clone())         # consumed by a torch op on the same stream
            del y
        got = torch.stack(outs).cpu().numpy()  # a copy on the same stream, no synchronize before it
    for row in got:
        assert rel_l2(row, ref) <= TOL64
    ex.close()


@pytest.mark.parametrize("cfg", ["c1", "c2"])
@pytest.mark.parametrize("kind", [K.windowed, K.gather, K.atomic, K.colorful, K.local_buffers])
def test_configs_full_size(cfg, kind):
    a, x, _ = P.config_matrix(cfg)
    ref = O.spmv_csrc(a, x)
    y = run(a, x, P.Strategy(kind, p=8))
    assert rel_l2(y, ref) <= TOL64 and rel_inf(y, ref) <= TOL64


# every kernel kind x accumulation, the kinds the north star names included
LARGE_KINDS = [
    ("gather", P.Strategy(K.gather)),
    ("windowed", P.Strategy(K.windowed)),
    ("atomic", P.Strategy(K.atomic)),
    ("colorful_nbh", P.Strategy(K.colorful, p=8)),
    ("colorful_exact", P.Strategy(K.colorful, p=8, conflict_mode=P.ConflictMode.exact)),
    ("lb_all_in_one", P.Strategy(K.local_buffers, A.all_in_one, p=8)),
    ("lb_per_buffer", P.Strategy(K.local_buffers, A.per_buffer, p=8)),
    ("lb_effective", P.Strategy(K.local_buffers, A.effective, p=8)),
    ("lb_interval", P.Strategy(K.local_buffers, A.interval, p=8)),
]
_big = {}


def big_config(cfg, f32=False):
    """(a, x, y_ref) for a BASELINE config, one config resident at a time. The
    oracle's full-size y is itself pinned to the reference's (sha256,
    tests/test_config_pins.py); fp32: the fp64 oracle on fp32-rounded inputs."""
    key = (cfg, f32)
    if key not in _big:
        _big.clear()
        a, x, _ = P.config_matrix(cfg)
        if f32:
            x = x.astype(np.float32).astype(np.float64)
            ref = O.spmv_csrc(round32(a), x)
        else:
            ref = O.spmv_csrc(a, x)
        _big[key] = (a, x, ref)
    return _big[key]


@pytest.mark.parametrize("name,s", LARGE_KINDS, ids=[n for n, _ in LARGE_KINDS])
@pytest.mark.parametrize("cfg", ["c3", "c4", "c5"])
def test_large_configs(cfg, name, s):
    a, x, ref = big_config(cfg)
    ex = P.GpuSpmv(a, s)
    try:
        y = ex.apply(x)
        assert rel_l2(y, ref) <= TOL64 and rel_inf(y, ref) <= TOL64, name
        if name.startswith("colorful"):
            assert ex.info().n_colors >= 2
        if name in ("gather", "windowed", "colorful_nbh", "lb_interval"):
            # linearity, a size-independent property: A(x + 2 z) = A x + 2 A z
            z = np.random.default_rng(1).uniform(-1, 1, a.n)
            lhs = ex.apply(x + 2 * z)
            rhs = ex.apply(x) + 2 * ex.apply(z)
            assert rel_l2(lhs, rhs) <= 1e-13
        if name in ("gather", "colorful_nbh"):
            assert np.array_equal(ex.apply(x), y)  # no atomics: bit-reproducible
    finally:
        ex.close()


@pytest.mark.parametrize("name,s", LARGE_KINDS, ids=[n for n, _ in LARGE_KINDS])
def test_c5_fp32(name, s):
    a, x32, ref = big_config("c5", f32=True)
    s32 = P.Strategy(s.kind, s.accum, p=s.p, dtype=P.DType.f32, conflict_mode=s.conflict_mode)
    y = run(a, x32, s32)
    assert rel_l2(y, ref) <= TOL32, name


@pytest.mark.parametrize("cfg", ["c3", "c5"])
def test_device_construction_matches_the_reference_at_scale(cfg):
    """build_csr -> csr_to_csrc (csr.hpp:55-92, csrc_matrix.hpp:44-91) on the
    device from the fixture's triplets in the golden shuffled order: the sha256
    of every CSRC array equals the reference's own construction of the same
    triplets (tests/golden/configs.json, made by oracle/_ref here)."""
    import hashlib
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "configs.json")) as f:
        g = json.load(f)
    gc = g["construction"][cfg]
    _big.clear()
    a, _, _ = P.config_matrix(cfg)
    n, _, r, c, v = P.csrc_to_triplets(a)
    perm = np.random.default_rng(g["shuffle_seed"]).permutation(r.size)
    r, c, v = r[perm], c[perm], v[perm]
    del perm
    assert r.size == gc["triplets"]
    b = P.build_csrc((n, n, r, c, v))
    del r, c, v
    assert b.value_symmetric == gc["value_symmetric"]
    for f in ("ad", "ia", "ja", "al", "au"):
        assert hashlib.sha256(np.ascontiguousarray(getattr(b, f)).tobytes()).hexdigest() == gc[f], f


@pytest.mark.parametrize("bands", [2, 3, 5])
@pytest.mark.parametrize("mesh", ["g1_", "g3_", "g5_"])
def test_band_plans_assemble_the_product(bands, mesh):
    """Multi-GPU decomposition on one device: each band's plan produces its
    owned rows plus the halo partial owed to lower bands; summing the halos
    into their owners (the NCCL exchange of paper_1003_0952_b200.dist)
    reproduces the full product."""
    import torch
    a = MESH.matrix(mesh)
    x = MESH[mesh + "x"]
    part = P.partition_by_nnz(a, bands)
    y = np.zeros(a.n)
    xd_full = torch.from_numpy(x).cuda()
    for b in range(bands):  # gather form: x over [lo, x_hi), own rows only, no exchange
        r0, r1 = part.begin(b), part.end(b)
        ex = P.GpuSpmv(a, P.Strategy(K.gather), band=(r0, r1))
        inf = ex.info()
        assert inf.lo <= r0 and inf.x_hi >= r1
        yd = torch.full((r1 - r0,), float("nan"), dtype=torch.float64, device="cuda")
        ex.apply_device(xd_full[inf.lo:inf.x_hi].contiguous(), yd)
        torch.cuda.synchronize()
        y[r0:r1] = yd.cpu().numpy()
        with pytest.raises(P.Error, match="partial products need the windowed kernel"):
            ex.apply_device_part(xd_full, yd, 0)
        ex.close()
    assert rel_l2(y, MESH[mesh + "y"]) <= TOL64
    y = np.zeros(a.n)
    for b in range(bands):
        r0, r1 = part.begin(b), part.end(b)
        ex = P.GpuSpmv(a, P.Strategy(K.windowed), band=(r0, r1))
        inf = ex.info()
        lo = inf.lo
        xd = xd_full[lo:r1].contiguous()
        yd = torch.zeros_like(xd)
        if b % 2 == 0:
            ex.apply_device(xd, yd)
        else:  # boundary rows first, then the interior (overlap form)
            ex.apply_device_part(xd, yd, 0)
            ex.apply_device_part(xd, yd, 1)
        torch.cuda.synchronize()
        y[lo:r1] += yd.cpu().numpy()
        assert ex.band_split() >= r0
        ex.close()
    assert rel_l2(y, MESH[mesh + "y"]) <= TOL64


@pytest.mark.parametrize("cfg", ["c2", "c4"])
@pytest.mark.parametrize("bands", [2, 3])
def test_gather_interior_rows_overlap_form(cfg, bands):
    """x-halo refresh form of the gather bands (dist.DistSpmv refresh_x): the
    interior rows run while the x halo is still garbage (NaN), the boundary
    rows after it lands; the result equals the one-shot band product bit for
    bit and the oracle."""
    import torch
    a, x, _ = P.config_matrix(cfg)
    ref = O.spmv_csrc(a, x)
    part = P.partition_by_nnz(a, bands)
    xd = torch.from_numpy(x).cuda()
    for b in range(bands):
        r0, r1 = part.begin(b), part.end(b)
        ex = P.GpuSpmv(a, P.Strategy(K.gather), band=(r0, r1))
        inf = ex.info()
        g0, g1 = ex.gather_interior()
        assert 0 <= g0 <= g1 <= r1 - r0 and g0 % 256 == 0
        assert g1 > g0, "bands of these meshes have interior rows"
        full = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
        xl = xd[inf.lo:inf.x_hi].contiguous()
        ex.apply_device(xl, full)
        halo = xl.clone()
        halo[: r0 - inf.lo] = float("nan")
        halo[r1 - inf.lo:] = float("nan")
        y = torch.full((r1 - r0,), float("nan"), dtype=torch.float64, device="cuda")
        ex.apply_device_rows(halo, y, g0, g1)
        torch.cuda.synchronize()
        assert not torch.isnan(y[g0:g1]).any()
        halo.copy_(xl)
        ex.apply_device_rows(halo, y, 0, g0)
        ex.apply_device_rows(halo, y, g1, r1 - r0)
        torch.cuda.synchronize()
        assert torch.equal(y, full)
        assert rel_l2(y.cpu().numpy(), ref[r0:r1]) <= TOL64
        with pytest.raises(P.Error, match="multiple of 256"):
            ex.apply_device_rows(halo, y, 1, g1)
        ex.close()
    ex = P.GpuSpmv(a, P.Strategy(K.windowed))
    with pytest.raises(P.Error, match="gather plan"):
        ex.apply_device_rows(xd, xd, 0, 256)
    ex.close()


@pytest.mark.parametrize("kind", ["gather", "windowed"])
def test_pageable_host_vectors(kind):
    """The host API stages pageable x / y (plain numpy here, std::vector in the
    reference's API) through pinned buffers: same bits as pinned vectors and
    as the device entry point, with y given, fresh, or a strided view."""
    import torch
    a, x, _ = P.config_matrix("c2")
    ex = P.GpuSpmv(a, P.Strategy(K[kind]))
    xh = torch.from_numpy(x.copy()).pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    ex.apply(xh.numpy(), yh.numpy())
    ref = yh.numpy().copy()
    y_page = np.empty(a.n)
    ex.apply(np.array(x), y_page)
    fresh = ex.apply(np.array(x))
    if kind == "gather":  # deterministic kernel: bit-identical across host paths
        assert np.array_equal(y_page, ref) and np.array_equal(fresh, ref)
    assert rel_l2(y_page, O.spmv_csrc(a, x)) <= TOL64 and rel_l2(fresh, ref) <= TOL64
    ex.close()


@pytest.mark.parametrize("cfg", ["c3", "c4"])
@pytest.mark.parametrize("env", [{}, {"CSRC_GPU_HOST_XHALO": "0"},
                                 {"CSRC_GPU_HOST_UNITS": "1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1"}])
def test_host_pipeline_matches_device(cfg, env, monkeypatch):
    """The host entry point of a gather plan overlaps the x upload, the row
    chunks and the y download (capi.cu apply_host_pipelined); it must give
    exactly the device entry point's result (same kernels, same order) with
    halo-aligned x chunks (default), row-aligned x chunks, and many small
    chunks (x chunks narrower than the halo: some come up empty)."""
    import torch
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    a, x, _ = P.config_matrix(cfg)
    ref = O.spmv_csrc(a, x)
    for dt, tdt in ((P.DType.f64, torch.float64), (P.DType.f32, torch.float32)):
        ex = P.GpuSpmv(a, P.Strategy(K.gather, dtype=dt))
        xd = torch.from_numpy(x).to(device="cuda", dtype=tdt)
        yd = torch.empty_like(xd)
        for tr in (False, True):
            yh = ex.apply(x, transpose=tr)
            ex.apply_device(xd, yd, transpose=tr)
            torch.cuda.synchronize()
            assert np.array_equal(yh, yd.double().cpu().numpy()), (dt, tr)
        if dt == P.DType.f64:
            assert rel_l2(ex.apply(x), ref) <= TOL64
        ex.close()


GATHER_SHAPES = [
    {"CSRC_GPU_GPATTERN": "0"},
    {"CSRC_GPU_GPATTERN": "0", "CSRC_GPU_GLANES": "4"},
    {"CSRC_GPU_GLANES": "8", "CSRC_GPU_GU": "8"},
    {"CSRC_GPU_GBUF": "0", "CSRC_GPU_GLANES": "1"},
    {"CSRC_GPU_GBUF": "0", "CSRC_GPU_GLANES": "4", "CSRC_GPU_GPF": "2"},
    {"CSRC_GPU_GBUF": "0", "CSRC_GPU_GLANES": "16"},
    {"CSRC_GPU_GNB": "2", "CSRC_GPU_GLANES": "2", "CSRC_GPU_GU": "8"},
    {"CSRC_GPU_GNB": "1", "CSRC_GPU_GLANES": "8", "CSRC_GPU_GU": "4"},
    {"CSRC_GPU_GNB": "1", "CSRC_GPU_GLANES": "16", "CSRC_GPU_GU": "8"},
    # row setup (eptr / pbase) staged with the values instead of global loads
    {"CSRC_GPU_GROWS": "1"},
    {"CSRC_GPU_GROWS": "1", "CSRC_GPU_GPATTERN": "0", "CSRC_GPU_GNB": "2"},
    {"CSRC_GPU_GROWS": "1", "CSRC_GPU_GLANES": "4", "CSRC_GPU_GNT": "128"},
    {"CSRC_GPU_GPATTERN": "0", "CSRC_GPU_GNB": "2", "CSRC_GPU_GNT": "64"},
    # staged, one row per thread
    {"CSRC_GPU_GLANES": "1"},
    {"CSRC_GPU_GLANES": "1", "CSRC_GPU_GPATTERN": "0", "CSRC_GPU_GNT": "128"},
    # sliced (SELL) form: lanes per row, steps in flight, pattern / explicit columns
    {"CSRC_GPU_GSELL": "1"},
    {"CSRC_GPU_GSELL": "1", "CSRC_GPU_SELL_L": "2"},
    {"CSRC_GPU_GSELL": "1", "CSRC_GPU_SELL_L": "4", "CSRC_GPU_SELL_U": "4"},
    {"CSRC_GPU_GSELL": "1", "CSRC_GPU_GPATTERN": "0", "CSRC_GPU_SELL_U": "12"},
    {"CSRC_GPU_GSELL": "1", "CSRC_GPU_SELL_U": "9"},
    {"CSRC_GPU_GSELL": "1", "CSRC_GPU_SELL_U": "14", "CSRC_GPU_SELL_L": "2"},
    {"CSRC_GPU_GSELL": "0"},
    # staged block sizes: 256 (the fp32 default), 128 (fp64 default), 64 threads
    {"CSRC_GPU_GNT": "256"},
    {"CSRC_GPU_GNT": "64"},
    {"CSRC_GPU_GNT": "128", "CSRC_GPU_GPATTERN": "0"},
]


@pytest.mark.parametrize("shape", range(len(GATHER_SHAPES)))
def test_gather_kernel_shapes(shape, monkeypatch):
    """Every gather kernel shape the plan can select (plain / staged, lanes,
    unroll, buffers; read from the environment at plan creation) gives the
    same bits as the default shape: the per-row summation order depends only
    on the lane count, so results are compared against the oracle and, for
    equal lane counts, bit for bit."""
    for k, v in GATHER_SHAPES[shape].items():
        monkeypatch.setenv(k, v)
    for idx in (0, 3, 5):
        p = f"g{idx}_"
        a = MESH.matrix(p)
        y = run(a, MESH[p + "x"], P.Strategy(K.gather))
        assert rel_l2(y, MESH[p + "y"]) <= TOL64
        yt = run(a, MESH[p + "x"], P.Strategy(K.gather), transpose=True)
        assert rel_l2(yt, O.spmv_csrc(a, MESH[p + "x"], transpose=True)) <= TOL64
    for idx in range(0, 29, 4):
        p = f"m{idx}_"
        a = FAM.matrix(p)
        assert rel_l2(run(a, FAM[p + "x"], P.Strategy(K.gather)), FAM[p + "y"]) <= TOL64


GATHER_SHAPES_F32 = [
    {},                                   # fp32 default: one row per thread, 6-block bound
    {"CSRC_GPU_GMINB": "1"},              # the unbounded one-row-per-thread form
    {"CSRC_GPU_GLANES": "2"},
    {"CSRC_GPU_GLANES": "3"},             # not instantiated: falls back to the default lanes
    {"CSRC_GPU_GLANES": "1", "CSRC_GPU_GPATTERN": "0"},
    {"CSRC_GPU_GSELL": "1"},
]


@pytest.mark.parametrize("shape", range(len(GATHER_SHAPES_F32)))
def test_gather_kernel_shapes_fp32(shape, monkeypatch):
    """fp32 gather shapes (the fp32-only defaults included) against the fp64
    oracle on fp32-rounded inputs."""
    for k, v in GATHER_SHAPES_F32[shape].items():
        monkeypatch.setenv(k, v)
    for idx in (0, 3, 5):
        p = f"g{idx}_"
        a = MESH.matrix(p)
        x32 = MESH[p + "x"].astype(np.float32).astype(np.float64)
        ref = O.spmv_csrc(round32(a), x32)
        y = run(a, x32, P.Strategy(K.gather, dtype=P.DType.f32))
        assert rel_l2(y, ref) <= TOL32


@pytest.mark.parametrize("dtype", [P.DType.f64, P.DType.f32])
def test_smaller_plan_does_not_break_a_live_larger_plan(dtype):
    """the dynamic shared-memory limit is an attribute of the
    kernel function that plans of one shape share. A large plan stays alive, a
    small plan of the same shape is created and run, then the large plan runs
    again and must still launch and match."""
    big, xb, _ = P.config_matrix("c2")
    small = MESH.matrix("g0_")
    ref_big = O.spmv_csrc(big, xb) if dtype == P.DType.f64 else O.spmv_csrc(
        round32(big), xb.astype(np.float32).astype(np.float64))
    xb_in = xb if dtype == P.DType.f64 else xb.astype(np.float32).astype(np.float64)
    tol = TOL64 if dtype == P.DType.f64 else TOL32
    for kind in (K.gather, K.windowed, K.local_buffers):
        ex_big = P.GpuSpmv(big, P.Strategy(kind, p=4, dtype=dtype))
        assert rel_l2(ex_big.apply(xb_in), ref_big) <= tol
        ex_small = P.GpuSpmv(small, P.Strategy(kind, p=4, dtype=dtype))
        ex_small.apply(MESH["g0_x"])
        assert rel_l2(ex_big.apply(xb_in), ref_big) <= tol, kind.name
        ex_small.close()
        ex_big.close()


@pytest.mark.parametrize("kind", [K.local_buffers, K.colorful, K.gather])
def test_mixing_plan_and_caller_streams(kind):
    """host apply() / time_products() run on the plan's own
    stream, apply_device on the caller's; a plan's scratch (band buffers, class-
    order vectors, timing events) is ordered across both."""
    import torch
    a, x, _ = P.config_matrix("c2")
    ref = O.spmv_csrc(a, x)
    ex = P.GpuSpmv(a, P.Strategy(kind, P.AccumMethod.interval, p=4))
    ex.set_timing(True)
    xd = torch.from_numpy(x).cuda()
    side = torch.cuda.Stream()
    outs = []
    for i in range(4):
        with torch.cuda.stream(side):
            yd = torch.full_like(xd, float("nan"))
            ex.apply_device(xd, yd)
            outs.append(yd)
        yh = ex.apply(x)  # plan stream, same scratch
        assert rel_l2(yh, ref) <= TOL64
        ex.time_products(xd, torch.empty_like(xd), 2)
    torch.cuda.synchronize()
    for yd in outs:
        assert rel_l2(yd.cpu().numpy(), ref) <= TOL64
    ex.close()


@pytest.mark.parametrize("lanes", ["1", "2", "4"])
def test_windowed_shared_memory_rings(lanes, monkeypatch):
    """The windowed kernel's optional shared-memory rings (CSRC_GPU_WIN_RINGS=1:
    in-window scatters resolved by CAS adds in shared memory, flushed with
    red.global; off by default because red.global alone is faster on B200)
    still give the product, also under the local-buffers accumulations and on
    band plans."""
    monkeypatch.setenv("CSRC_GPU_WIN_RINGS", "1")
    monkeypatch.setenv("CSRC_GPU_LANES", lanes)
    for idx in (1, 2, 3, 5):
        p = f"g{idx}_"
        a = MESH.matrix(p)
        ex = P.GpuSpmv(a, P.Strategy(K.windowed))
        assert ex.info().captured_fraction > 0
        assert rel_l2(ex.apply(MESH[p + "x"]), MESH[p + "y"]) <= TOL64
        ex.close()
        for acc in (A.effective, A.interval):
            y = run(a, MESH[p + "x"], P.Strategy(K.local_buffers, acc, p=4))
            assert rel_l2(y, MESH[p + "y"]) <= TOL64
    for idx in range(0, 29, 7):
        p = f"m{idx}_"
        a = FAM.matrix(p)
        assert rel_l2(run(a, FAM[p + "x"], P.Strategy(K.windowed)), FAM[p + "y"]) <= TOL64


@pytest.mark.parametrize("lanes", ["1", "2"])
def test_sliced_form_bands_pipeline_and_bits(lanes, monkeypatch):
    """The sliced gather form (k_gather_sell) on band plans, through the host
    pipeline (row chunks = whole slices) and with explicit columns: the same
    bits as the pattern form, oracle parity for y and y^T."""
    import torch
    monkeypatch.setenv("CSRC_GPU_GSELL", "1")
    monkeypatch.setenv("CSRC_GPU_SELL_L", lanes)
    a = MESH.matrix("g2_")
    x = MESH["g2_x"]
    ex = P.GpuSpmv(a, P.Strategy(K.gather))
    assert ex.info().gather_form == 3
    y = ex.apply(x)
    yt = ex.apply(x, transpose=True)
    ex.close()
    assert rel_l2(y, MESH["g2_y"]) <= TOL64
    assert rel_l2(yt, O.spmv_csrc(a, x, transpose=True)) <= TOL64
    monkeypatch.setenv("CSRC_GPU_GPATTERN", "0")
    ex = P.GpuSpmv(a, P.Strategy(K.gather))
    assert ex.info().row_patterns == 0 and ex.info().gather_form == 3
    assert np.array_equal(ex.apply(x), y)
    ex.close()
    part = P.partition_by_nnz(a, 3)
    yb = np.zeros(a.n)
    xd = torch.from_numpy(x).cuda()
    for b in range(3):
        r0, r1 = part.begin(b), part.end(b)
        eb = P.GpuSpmv(a, P.Strategy(K.gather), band=(r0, r1))
        inf = eb.info()
        yd = torch.empty(r1 - r0, dtype=torch.float64, device="cuda")
        eb.apply_device(xd[inf.lo:inf.x_hi].contiguous(), yd)
        torch.cuda.synchronize()
        yb[r0:r1] = yd.cpu().numpy()
        eb.close()
    assert rel_l2(yb, MESH["g2_y"]) <= TOL64


def test_gather_dense_row_falls_back():
    """An arrow matrix whose first column is full: row 0's entry stream (every
    other row names it) does not fit a shared-memory row block, so the plan
    takes the plain row kernel; results still match the oracle."""
    n = 40000
    rng = np.random.default_rng(5)
    ia = np.zeros(n + 1, np.int32)
    ia[1:] = np.arange(n, dtype=np.int32)  # row r >= 1 stores the single pair (r, 0)
    ja = np.zeros(n - 1, np.int32)
    al = rng.uniform(-1, 1, n - 1)
    au = rng.uniform(-1, 1, n - 1)
    ad = 4 + rng.uniform(0, 1, n)
    a = P.CsrcMatrix(n, ad, ia, ja, al, au)
    x = rng.uniform(-1, 1, n)
    for kind in (K.gather, K.sequential):
        y = run(a, x, P.Strategy(kind))
        assert rel_l2(y, O.spmv_csrc(a, x)) <= TOL64
        assert rel_l2(run(a, x, P.Strategy(kind), transpose=True), O.spmv_csrc(a, x, transpose=True)) <= TOL64


@pytest.mark.parametrize("cfg", ["c2", "c4"])
def test_row_patterns_are_bit_identical(cfg, monkeypatch):
    """Mesh matrices repeat a few column-offset patterns: the gather plan
    stores a pattern start per row instead of a column index per entry
    (k_gather_staged<PAT>); same entry order, so the same bits as the
    explicit-index form, and the plan reports the dictionary size."""
    a, x, _ = P.config_matrix(cfg)
    ex = P.GpuSpmv(a, P.Strategy(K.gather))
    inf = ex.info()
    assert 0 < inf.row_patterns <= 200, inf.row_patterns
    assert inf.stream_bytes < inf.model_bytes
    y_pat = ex.apply(x)
    yt_pat = ex.apply(x, transpose=True)
    ex.close()
    monkeypatch.setenv("CSRC_GPU_GPATTERN", "0")
    ex = P.GpuSpmv(a, P.Strategy(K.gather))
    assert ex.info().row_patterns == 0
    assert np.array_equal(ex.apply(x), y_pat)
    assert np.array_equal(ex.apply(x, transpose=True), yt_pat)
    ex.close()
    assert rel_l2(y_pat, O.spmv_csrc(a, x)) <= TOL64


def test_permuted_mesh_has_no_small_dictionary():
    """C3 is randomly permuted then RCM-ordered: rows do not repeat offsets,
    the plan keeps explicit indices."""
    a, x, _ = P.config_matrix("c3")
    ex = P.GpuSpmv(a, P.Strategy(K.gather))
    assert ex.info().row_patterns == 0
    ex.close()


COLORED_SHAPES = [
    {},                                                                   # ring form, defaults
    {"CSRC_GPU_CW_RING": "0"},                                            # direct wavefront (no TMA ring)
    {"CSRC_GPU_COLOR_WAVE": "0"},                                         # one launch per class
    {"CSRC_GPU_CR_STAGE_BYTES": "2560", "CSRC_GPU_CW_U": "4"},            # 1-pair sub-chunks: many fills per chunk
    {"CSRC_GPU_CR_STAGE_BYTES": "7680", "CSRC_GPU_CR_STAGES": "3", "CSRC_GPU_CW_U": "8"},
    {"CSRC_GPU_CR_STAGES": "6", "CSRC_GPU_CW_U": "16"},
    {"CSRC_GPU_CR_HINT": "1"},                                            # evict_last on the x / y window
    {"CSRC_GPU_CW_R": "1", "CSRC_GPU_CW_D": "2"},                         # tightest dependency distance
    {"CSRC_GPU_CW_R": "8", "CSRC_GPU_CW_MINB": "1"},                      # many small blocks, radius 8
    {"CSRC_GPU_CW_CTAS": "1"},                                            # one CTA per SM
    {"CSRC_GPU_CR_SPLIT": "1", "CSRC_GPU_CW_U": "14"},                    # setmaxnreg register split
    {"CSRC_GPU_CR_PF": "1", "CSRC_GPU_CR_STAGES": "3"},                   # L2 prefetcher warp
    {"CSRC_GPU_CR_PF": "1", "CSRC_GPU_CR_STAGE_BYTES": "5120", "CSRC_GPU_CW_U": "4"},
    {"CSRC_GPU_CR_LANES": "2"},                                           # two lanes per row, 64-row chunks
    {"CSRC_GPU_CR_LANES": "2", "CSRC_GPU_CR_STAGE_BYTES": "3840", "CSRC_GPU_CR_STAGES": "4"},
    {"CSRC_GPU_CR_CLAIM": "1"},                                           # loader claims after staging
    {"CSRC_GPU_CR_CLAIM": "2", "CSRC_GPU_CR_STAGES": "3", "CSRC_GPU_CR_SLACK_PCT": "100"},
]


@pytest.mark.parametrize("env", COLORED_SHAPES, ids=lambda e: ",".join(f"{k[9:]}={v}" for k, v in e.items()) or "default")
def test_colored_kernel_shapes(env, monkeypatch):
    """Every form / shape of the colored kernel (colored.cuh): the TMA-ring
    wavefront (default), the direct wavefront and the launch-per-class form,
    with stage sizes that split chunks into many sub-chunks, every U, deep and
    shallow rings, tight and wide dependency windows -- y and y^T against the
    oracle on the golden meshes (fp64 and fp32), bit-identical repeats (no
    atomics), and the reference's class-order result on the family."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for key in ("g1_", "g2_", "g3_", "g4_"):
        a = MESH.matrix(key)
        x = MESH[key + "x"]
        for mode in (P.ConflictMode.neighborhood, P.ConflictMode.exact):
            ex = P.GpuSpmv(a, P.Strategy(K.colorful, p=4, conflict_mode=mode))
            y = ex.apply(x)
            assert rel_l2(y, MESH[key + "y"]) <= TOL64, (key, mode)
            assert np.array_equal(ex.apply(x), y), (key, mode)
            assert rel_l2(ex.apply(x, transpose=True), O.spmv_csrc(a, x, transpose=True)) <= TOL64, (key, mode)
            ex.close()
        x32 = x.astype(np.float32).astype(np.float64)
        y32 = run(a, x32, P.Strategy(K.colorful, p=4, dtype=P.DType.f32))
        assert rel_l2(y32, O.spmv_csrc(round32(a), x32)) <= TOL32, key
    for idx in (0, 7, 19, 25, 28):
        p = f"m{idx}_"
        a = FAM.matrix(p)
        assert rel_l2(run(a, FAM[p + "x"], P.Strategy(K.colorful, p=3)), FAM[p + "y"]) <= TOL64, idx
