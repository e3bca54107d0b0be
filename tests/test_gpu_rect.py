"""Rectangular CSRC products (CsrcRectMatrix, csrc_matrix.hpp:35-39;
spmv_csrc_rect kernels.hpp:69-91; ParallelSpmv over a rect matrix
parallel.hpp:168-181, 300-304) on the GPU against the oracle and the compiled
reference. Bar: fp64 relative L2 <= 1e-12 (and the reference's inf-norm check),
fp32 <= 1e-5 against the fp64 oracle on fp32-rounded inputs."""
import numpy as np
import pytest

import paper_1003_0952_b200 as P
from oracle.oracle import Oracle, Ref
from tests.helpers import family, meshes, rel_inf, rel_l2

pytestmark = pytest.mark.gpu
K = P.StrategyKind


def make_rect(a, extra, per_row, seed):
    rng = np.random.default_rng(seed)
    cnt = rng.integers(0, per_row + 1, a.n)
    rp = np.r_[0, np.cumsum(cnt)].astype(np.int32)
    ci = np.concatenate([np.sort(rng.choice(extra, size=int(c), replace=False)) for c in cnt]).astype(np.int32) \
        if cnt.sum() else np.zeros(0, np.int32)
    va = rng.uniform(-1, 1, int(cnt.sum()))
    return P.CsrcRectMatrix(a, P.CsrMatrix(a.n, extra, rp, ci, va), a.n + extra)


STRATS = [
    P.Strategy(K.gather), P.Strategy(K.sequential), P.Strategy(K.windowed), P.Strategy(K.atomic),
    P.Strategy(K.colorful, p=4),
    *[P.Strategy(K.local_buffers, m, p=3) for m in P.AccumMethod],
]


@pytest.mark.parametrize("si", range(len(STRATS)))
def test_rect_family_all_kinds(si):
    s = STRATS[si]
    fam = family()
    O, R = Oracle(), Ref()
    for idx in (0, 5, 11, 26):
        a = fam.matrix(f"m{idx}_")
        r = make_rect(a, 23, 4, idx)
        x = np.random.default_rng(idx).uniform(-1, 1, r.m)
        ref = R.spmv_csrc_rect(r, x)
        assert rel_l2(O.spmv_csrc_rect(r, x), ref) <= 1e-15
        y = P.GpuSpmv(r, s).apply(x)
        assert rel_l2(y, ref) <= 1e-12 and rel_inf(y, ref) <= 1e-12, (s, idx)


def test_rect_mesh_f32_and_device_path():
    a = meshes().matrix("g1_")
    r = make_rect(a, 101, 6, 3)
    x = np.random.default_rng(1).uniform(-1, 1, r.m)
    ref = Ref().spmv_csrc_rect(r, x)
    assert rel_l2(P.spmv_csrc_rect(r, x), ref) <= 1e-12
    r32 = P.CsrcRectMatrix(
        P.CsrcMatrix(a.n, a.ad.astype(np.float32).astype(np.float64), a.ia, a.ja,
                     a.al.astype(np.float32).astype(np.float64), a.au.astype(np.float32).astype(np.float64)),
        P.CsrMatrix(a.n, 101, r.rect.row_ptr, r.rect.col_idx, r.rect.values.astype(np.float32).astype(np.float64)),
        r.m)
    x32 = x.astype(np.float32).astype(np.float64)
    ref32 = Oracle().spmv_csrc_rect(r32, x32)
    for kind in (K.gather, K.windowed, K.atomic):
        y = P.GpuSpmv(r32, P.Strategy(kind, dtype=P.DType.f32)).apply(x32)
        assert rel_l2(y, ref32) <= 1e-5
    import torch
    ex = P.GpuSpmv(r, P.Strategy(K.gather))
    dx = torch.tensor(x, device="cuda")
    dy = torch.empty(a.n, dtype=torch.float64, device="cuda")
    ex.apply_device(dx, dy)
    torch.cuda.synchronize()
    assert rel_l2(dy.cpu().numpy(), ref) <= 1e-12
    assert ex.info().m_cols == r.m and ex.info().rect_nnz == r.rect.nnz()


def test_rect_errors():
    a = meshes().matrix("g0_")
    r = make_rect(a, 5, 2, 0)
    ex = P.GpuSpmv(r, P.Strategy(K.gather))
    with pytest.raises(P.Error, match=f"ParallelSpmv: x has length {a.n}, expected {a.n + 5}"):
        ex.apply(np.zeros(a.n))
    with pytest.raises(P.Error, match="no transpose product"):
        ex.apply(np.zeros(r.m), transpose=True)
    bad = P.CsrcRectMatrix(a, P.CsrMatrix(a.n, 5, r.rect.row_ptr, r.rect.col_idx + 9, r.rect.values), r.m)
    if r.rect.nnz():
        with pytest.raises(P.Error, match="rect tail: column"):
            P.GpuSpmv(bad, P.Strategy(K.gather))


def test_rect_from_decompose_rect():
    """CSR n x m -> decompose_rect on the device -> rect product == reference
    spmv_csrc_rect of the reference's own decomposition."""
    a = meshes().matrix("g2_")
    n, _, r, c, v = P.csrc_to_triplets(a)
    rng = np.random.default_rng(9)
    tr = rng.integers(0, n, 3 * n).astype(np.int32)
    tc = (n + rng.integers(0, 64, 3 * n)).astype(np.int32)
    R = Ref()
    rp, ci, va = R.build_csr(n, n + 64, np.r_[r, tr], np.r_[c, tc], np.r_[v, rng.uniform(-1, 1, 3 * n)])
    sq, (trp, tci, tva) = R.decompose_rect(n, n + 64, rp, ci, va)
    ref_rect = P.CsrcRectMatrix(P.CsrcMatrix(**sq), P.CsrMatrix(n, 64, trp, tci, tva), n + 64)
    got = P.decompose_rect(P.CsrMatrix(n, n + 64, rp, ci, va))
    x = rng.uniform(-1, 1, n + 64)
    ref = R.spmv_csrc_rect(ref_rect, x)
    for kind in (K.gather, K.windowed, K.colorful):
        s = P.Strategy(kind, p=2 if kind == K.colorful else 1)
        assert rel_l2(P.GpuSpmv(got, s).apply(x), ref) <= 1e-12
