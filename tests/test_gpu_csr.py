"""spmv_csr (kernels.hpp:7-22) on the GPU: general CSR plans
(csrc_gpu_plan_create_csr) against the compiled reference's spmv_csr, on the
reference's generator family (full CSR of each CSRC matrix), on rectangular
and pattern-unsymmetric matrices, through every gather kernel form."""
import numpy as np
import pytest

import paper_1003_0952_b200 as P
from oracle.oracle import Oracle, Ref
from tests.helpers import family, meshes, rel_inf, rel_l2

pytestmark = pytest.mark.gpu


def full_csr(a):
    n, _, r, c, v = P.csrc_to_triplets(a)
    rp, ci, va = Ref().build_csr(n, n, r, c, v)
    return P.CsrMatrix(n, n, rp, ci, va)


def random_csr(rng, n_rows, n_cols, per_row):
    cnt = rng.integers(0, per_row + 1, n_rows)
    rp = np.r_[0, np.cumsum(cnt)].astype(np.int32)
    ci = np.concatenate([np.sort(rng.choice(n_cols, int(c), replace=False)) for c in cnt]).astype(np.int32) \
        if cnt.sum() else np.zeros(0, np.int32)
    return P.CsrMatrix(n_rows, n_cols, rp, ci, rng.uniform(-1, 1, int(cnt.sum())))


FORMS = [{}, {"CSRC_GPU_GSELL": "1"}, {"CSRC_GPU_GPATTERN": "0"}, {"CSRC_GPU_GBUF": "0"},
         {"CSRC_GPU_GNT": "256"}]


@pytest.mark.parametrize("form", range(len(FORMS)))
def test_csr_family_and_meshes(form, monkeypatch):
    for k, v in FORMS[form].items():
        monkeypatch.setenv(k, v)
    R = Ref()
    fam = family()
    for idx in range(0, 29, 3):
        a = fam.matrix(f"m{idx}_")
        m = full_csr(a)
        x = fam[f"m{idx}_x"]
        ref = R.spmv_csr(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values, x)
        y = P.spmv_csr(m, x)
        assert rel_l2(y, ref) <= 1e-12 and rel_inf(y, ref) <= 1e-12
        assert rel_l2(y, Oracle().spmv_csrc(a, x)) <= 1e-12
    for g in range(4):
        a = meshes().matrix(f"g{g}_")
        m = full_csr(a)
        assert rel_l2(P.spmv_csr(m, meshes()[f"g{g}_x"]), meshes()[f"g{g}_y"]) <= 1e-12


@pytest.mark.parametrize("shape", [(1000, 700), (700, 1000), (4096, 4096), (3, 50000)])
def test_csr_rectangular_and_unsymmetric(shape):
    rng = np.random.default_rng(shape[0] + shape[1])
    m = random_csr(rng, shape[0], shape[1], 9)
    x = rng.uniform(-1, 1, shape[1])
    ref = Ref().spmv_csr(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values, x)
    ex = P.GpuSpmv(m, P.Strategy(P.StrategyKind.gather))
    assert ex.info().csr_cols == shape[1]
    y = ex.apply(x)
    assert rel_l2(y, ref) <= 1e-12
    m32 = P.CsrMatrix(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values.astype(np.float32).astype(np.float64))
    x32 = x.astype(np.float32).astype(np.float64)
    ref32 = Ref().spmv_csr(m.n_rows, m.n_cols, m32.row_ptr, m32.col_idx, m32.values, x32)
    y32 = P.GpuSpmv(m32, P.Strategy(P.StrategyKind.gather, dtype=P.DType.f32)).apply(x32)
    assert rel_l2(y32, ref32) <= 1e-5


def test_csr_host_pipeline_and_device_bits():
    import torch
    a, x, _ = P.config_matrix("c2")
    m = full_csr(a)
    ex = P.GpuSpmv(m, P.Strategy(P.StrategyKind.gather))
    yh = ex.apply(x)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    ex.apply_device(xd, yd)
    torch.cuda.synchronize()
    assert np.array_equal(yh, yd.cpu().numpy())
    assert rel_l2(yh, Oracle().spmv_csrc(a, x)) <= 1e-12
    assert ex.info().row_patterns > 0  # the full 27-point rows repeat a small dictionary


def test_csr_errors():
    m = P.CsrMatrix(3, 4, np.array([0, 1, 2, 2], np.int32), np.array([0, 3], np.int32), np.array([1.0, 2.0]))
    with pytest.raises(P.Error, match="spmv_csr: x has length 3, expected 4"):
        P.spmv_csr(m, np.zeros(3))
    ex = P.GpuSpmv(m, P.Strategy(P.StrategyKind.gather))
    with pytest.raises(P.Error, match="no transpose product"):
        ex.apply(np.zeros(4), transpose=True)
    assert P.spmv_csr(m, np.array([1.0, 0, 0, 5.0])).tolist() == [1.0, 10.0, 0.0]
    bad = P.CsrMatrix(2, 2, np.array([0, 1, 2], np.int32), np.array([0, 2], np.int32), np.array([1.0, 1.0]))
    with pytest.raises(P.Error, match="column 2 outside"):
        P.GpuSpmv(bad, P.Strategy(P.StrategyKind.gather))
    with pytest.raises(P.Error, match="sequential or gather"):
        P.GpuSpmv(m, P.Strategy(P.StrategyKind.windowed))
