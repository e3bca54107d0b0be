"""The product's direct CSRC fixture assembly (fixtures/csrc_fixtures.cpp) equals the
reference pipeline build_csr -> csr_to_csrc applied to the restated mesh
entries: golden vectors (reference output) for small meshes, live reference
(oracle/_ref) for C1 and C2 at full size when it is present."""
import numpy as np
import pytest

from oracle.oracle import Oracle, Ref, mesh_triplets

import paper_1003_0952_b200 as P

from .helpers import meshes

MESH = meshes()


@pytest.mark.parametrize("idx", range(6))
def test_fixture_generator_matches_reference_construction(idx):
    p = f"g{idx}_"
    mesh, nx, ny, nz, seed = (int(v) for v in MESH[p + "spec"])
    a, x, order = P.generate_fixture(P.Mesh(mesh), nx, ny, nz, seed, float(MESH[p + "diag"]))
    for k in ("ad", "ia", "ja", "al", "au"):
        assert np.array_equal(getattr(a, k), MESH[p + k]), k
    assert np.array_equal(x, MESH[p + "x"])
    assert np.array_equal(order, MESH[p + "order"])


def test_fixture_thread_count_does_not_change_the_matrix():
    a1, x1, _ = P.generate_fixture(P.Mesh.grid3d_27_rcm, 7, 6, 5, 11, 30.0, threads=1)
    a8, x8, _ = P.generate_fixture(P.Mesh.grid3d_27_rcm, 7, 6, 5, 11, 30.0, threads=8)
    for k in ("ad", "ia", "ja", "al", "au"):
        assert np.array_equal(getattr(a1, k), getattr(a8, k))
    assert np.array_equal(x1, x8)


@pytest.mark.parametrize("name,n,nnz,k", [
    ("c1", 65536, 586756, 260610),
    ("c2", 262144, 6859000, 3298428),
])
def test_config_sizes(name, n, nnz, k):
    a, x, _ = P.config_matrix(name)
    assert a.n == n and a.nnz_full() == nnz and a.k_off() == k
    assert not a.value_symmetric
    c = P.CONFIGS[name]
    assert np.all(a.ad >= c["diag_base"]) and np.all(a.ad < c["diag_base"] + 1)
    assert np.all(np.abs(a.al) <= 1) and np.all(np.abs(x) <= 1)


@pytest.mark.skipif(not Ref.available(), reason="reference shim oracle/_ref not built here")
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_config_construction_matches_live_reference(name):
    c = P.CONFIGS[name]
    a, x, order = P.config_matrix(name)
    n, r, cc, v, xo, oo = mesh_triplets(int(c["mesh"]), c["nx"], c["ny"], c["nz"], c["seed"], c["diag_base"])
    ref = Ref().build_csrc(n, r, cc, v)
    for k in ("ad", "ia", "ja", "al", "au"):
        assert np.array_equal(getattr(a, k), ref[k]), k
    assert np.array_equal(x, xo)


def test_rcm_fixture_is_a_symmetric_permutation():
    """P A P^T of the natural matrix: same multiset of entries, and the RCM
    order narrows the bandwidth of the randomly permuted graph."""
    nat, _, _ = P.generate_fixture(P.Mesh.grid3d_27, 10, 9, 8, 11, 30.0)
    rcm, _, order = P.generate_fixture(P.Mesh.grid3d_27_rcm, 10, 9, 8, 11, 30.0)
    assert rcm.k_off() == nat.k_off() and np.array_equal(np.sort(order), np.arange(rcm.n))
    assert np.array_equal(np.sort(np.concatenate([rcm.al, rcm.au])), np.sort(np.concatenate([nat.al, nat.au])))
    bw = max(int(i - rcm.ja[rcm.ia[i]]) for i in range(rcm.n) if rcm.ia[i + 1] > rcm.ia[i])
    assert bw < rcm.n // 3


def test_oracle_spmv_on_config_c1():
    a, x, _ = P.config_matrix("c1")
    y = Oracle().spmv_csrc(a, x)
    assert y.shape == (a.n,) and np.isfinite(y).all()


@pytest.mark.parametrize("mesh,dims", [(0, (9, 7, 1)), (1, (6, 5, 4)), (2, (4, 3, 5)), (3, (7, 6, 5))])
def test_standalone_fixture_library_equals_the_product_generator(mesh, dims):
    """oracle/_build/libcsrc_fixtures.so (the reference arm's input generator)
    and the product library build the same matrices from the same source."""
    from oracle.oracle import fixture
    a, x, _ = P.generate_fixture(P.Mesh(mesh), *dims, 5, 30.0)
    b, xb = fixture(mesh, *dims, 5, 30.0)
    for f in ("ad", "ia", "ja", "al", "au"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(x, xb)
