"""Pins the plain-C oracle (oracle/csrc_oracle.c) to the reference: every
known answer of the reference's own tests and the golden vectors produced by
running the reference itself (tests/golden/make_golden.py). Where the compiled
reference (oracle/_ref) is present, also cross-checks live on fresh inputs."""
import numpy as np
import pytest

from oracle.oracle import Oracle, Ref, mesh_triplets, u01 as np_u01

import paper_1003_0952_b200 as P

from .helpers import family, known_answers, matrix_from_dict, meshes

O = Oracle()
KA = known_answers()
FAM = family()
MESH = meshes()


def test_known_answer_spmv():
    for key in ("spmv_diag", "spmv_2x2"):
        ka = KA[key]
        a = matrix_from_dict(ka["matrix"])
        assert O.spmv_csrc(a, ka["x"]).tolist() == ka["y"]


def test_known_answer_2x2_local_buffers():
    ka = KA["spmv_2x2"]
    a = matrix_from_dict(ka["matrix"])
    assert O.spmv_local_buffers(a, ka["x"], ka["block_start"]).tolist() == ka["y"]


def test_known_answer_partition():
    ka = KA["partition_counts"]
    a = matrix_from_dict(ka["matrix"])
    bs, bn = O.partition_by_nnz(a, ka["p"])
    assert bs == ka["block_start"] and bn == ka["block_nnz"]


def test_known_answer_effective_ranges():
    for case in KA["effective_ranges"]["cases"]:
        a = matrix_from_dict(case["matrix"])
        lo, hi = O.effective_ranges(a, case["block_start"])
        assert lo == case["lo"] and hi == case["hi"]


def test_known_answer_interval_plans():
    for case in KA["interval_plans"]["cases"]:
        bd, ivs = O.interval_plan(case["lo"], case["hi"])
        assert bd == case["boundaries"]
        assert [list(map(lambda v: v if not isinstance(v, tuple) else list(v), iv)) for iv in ivs] == \
               [[b, e, c] for b, e, c in case["intervals"]]


def test_known_answer_tridiagonal_coloring():
    ka = KA["tridiag4_coloring"]
    a = matrix_from_dict(ka["matrix"])
    for mode, key in ((0, "neighborhood"), (1, "exact")):
        col, nc = O.color_rows(a, mode, 0)
        assert col.tolist() == ka[key]["color"] and nc == ka[key]["n_colors"]
        assert list(O.conflict_edge_counts(a, mode)) == ka[key]["edges"]


def test_known_answer_coloring_violation():
    ka = KA["coloring_violation"]
    a = matrix_from_dict(KA["tridiag4_coloring"]["matrix"])
    assert O.validate_coloring(a, ka["color"], ka["n_colors"]) == (False, 0, 1, 0)


def test_known_answer_working_set_and_ops():
    for n, nnz, vs, kb in KA["working_set_kb"]["rows"]:
        assert O.working_set_bytes(n, nnz, vs) // 1024 == kb
    for i, fmt in enumerate(["csr", "csrc", "csrc_sym"]):
        assert list(O.count_ops(i, 9, 33)) == KA["count_ops"]["flops_loads"][fmt]


@pytest.mark.parametrize("idx", range(29))
def test_family_spmv_bit_exact(idx):
    p = f"m{idx}_"
    a = FAM.matrix(p)
    # the restatement follows the reference FP order exactly: bit-identical
    assert np.array_equal(O.spmv_csrc(a, FAM[p + "x"]), FAM[p + "y"])
    assert np.array_equal(O.spmv_csrc(a, FAM[p + "xr"]), FAM[p + "yr"])
    assert np.array_equal(O.spmv_csrc(a, FAM[p + "xr"], transpose=True), FAM[p + "yt"])


@pytest.mark.parametrize("idx", range(29))
def test_family_plans(idx):
    p = f"m{idx}_"
    a = FAM.matrix(p)
    for pp in (1, 2, 3, 4, 8):
        if not FAM.has(p + f"p{pp}_bs"):
            continue
        bs, bn = O.partition_by_nnz(a, pp)
        assert bs == FAM[p + f"p{pp}_bs"].tolist() and bn == FAM[p + f"p{pp}_bn"].tolist()
        lo, hi = O.effective_ranges(a, bs)
        assert lo == FAM[p + f"p{pp}_lo"].tolist() and hi == FAM[p + f"p{pp}_hi"].tolist()
        bd, ivs = O.interval_plan(lo, hi)
        assert bd == FAM[p + f"p{pp}_bd"].tolist()
        assert [[b, e] for b, e, _ in ivs] == FAM[p + f"p{pp}_iv"].tolist()
        assert [len(c) for _, _, c in ivs] == FAM[p + f"p{pp}_ivc"].tolist()
        # local-buffers result within the reference tolerance (acceptance.cpp:214-266)
        y = O.spmv_local_buffers(a, FAM[p + "x"], bs)
        ref = FAM[p + "y"]
        assert np.max(np.abs(y - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1.0)


@pytest.mark.parametrize("idx", [i for i in range(29)])
def test_family_colorings(idx):
    p = f"m{idx}_"
    if not FAM.has(p + "col00"):
        pytest.skip("no colouring stored")
    a = FAM.matrix(p)
    if a.n > 200:
        pytest.skip("dense-matrix oracle colouring kept to n <= 200")
    for mode in (0, 1):
        assert list(O.conflict_edge_counts(a, mode)) == FAM[p + f"edges{mode}"].tolist()
        for order in (0, 1, 2):
            col, nc = O.color_rows(a, mode, order)
            assert col.tolist() == FAM[p + f"col{mode}{order}"].tolist()
            assert nc == int(FAM[p + f"nc{mode}{order}"])
            assert O.validate_coloring(a, col, nc)[0]


@pytest.mark.parametrize("idx", range(6))
def test_mesh_construction_matches_reference(idx):
    """oracle build_csr -> csr_to_csrc of the restated mesh entries equals
    the reference's construction (golden), bit for bit."""
    p = f"g{idx}_"
    mesh, nx, ny, nz, seed = (int(v) for v in MESH[p + "spec"])
    n, r, c, v, x, order = mesh_triplets(mesh, nx, ny, nz, seed, float(MESH[p + "diag"]))
    d = O.build_csrc(n, r, c, v)
    for k in ("ad", "ia", "ja", "al", "au"):
        assert np.array_equal(d[k], MESH[p + k]), k
    assert np.array_equal(x, MESH[p + "x"]) and np.array_equal(order, MESH[p + "order"])
    a = MESH.matrix(p)
    assert np.array_equal(O.spmv_csrc(a, x), MESH[p + "y"])


def test_construction_rejects_like_the_reference():
    with pytest.raises(ValueError, match=r"entry \(1, 0\) has no transpose \(0, 1\)"):
        O.build_csrc(2, [0, 1, 1], [0, 0, 1], [1.0, 2.0, 1.0])
    with pytest.raises(ValueError, match="row 1 has no diagonal entry"):
        O.build_csrc(2, [0], [0], [1.0])
    with pytest.raises(ValueError, match="outside 2x2 bounds"):
        O.build_csrc(2, [0, 2], [0, 0], [1.0, 1.0])


def test_fixture_hash_numpy_equals_c():
    rng = np.random.default_rng(0)
    for _ in range(200):
        s, a, b = (int(v) for v in rng.integers(0, 2**40, 3))
        assert np_u01(s, a, b) == P.fixture_u01(s, a, b)


@pytest.mark.skipif(not Ref.available(), reason="reference shim oracle/_ref not built here")
def test_oracle_matches_live_reference_on_fresh_matrices():
    R = Ref()
    for i in range(12):
        n = 30 + 37 * i
        r, c, v = R.gen_random_sym(n, 0.02 + 0.03 * (i % 5), 777 + i, i % 4 == 0)
        ref = R.build_csrc(n, r, c, v)
        mine = O.build_csrc(n, r, c, v)
        for k in ("ad", "ia", "ja", "al", "au"):
            assert np.array_equal(ref[k], mine[k])
        a = P.CsrcMatrix(n, ref["ad"], ref["ia"], ref["ja"], ref["al"], ref["au"], ref["value_symmetric"])
        x = np.random.default_rng(i).uniform(-1, 1, n)
        assert np.array_equal(O.spmv_csrc(a, x), R.spmv_csrc(a, x))


@pytest.mark.skipif(not Ref.available(), reason="reference shim oracle/_ref not built here")
def test_oracle_rect_product_bit_exact():
    """oracle_spmv_csrc_rect restates spmv_csrc_rect (kernels.hpp:69-91) in the
    reference's FP order: bit-identical on the family plus random CSR tails."""
    R = Ref()
    rng = np.random.default_rng(3)
    for idx in (0, 7, 19, 28):
        a = FAM.matrix(f"m{idx}_")
        extra = 11 + idx
        cnt = rng.integers(0, 4, a.n)
        rp = np.r_[0, np.cumsum(cnt)].astype(np.int32)
        ci = np.concatenate([np.sort(rng.choice(extra, int(c), replace=False)) for c in cnt]).astype(np.int32)
        r = P.CsrcRectMatrix(a, P.CsrMatrix(a.n, extra, rp, ci, rng.uniform(-1, 1, int(cnt.sum()))), a.n + extra)
        x = rng.uniform(-1, 1, r.m)
        assert np.array_equal(O.spmv_csrc_rect(r, x), R.spmv_csrc_rect(r, x))


def test_csrc_to_triplets_order():
    """P.csrc_to_triplets emits csrc_to_csr's triplet order (csrc_matrix.hpp:95-108)
    and the oracle's build_csr -> csr_to_csrc inverts it bit for bit."""
    a = MESH.matrix("g0_")
    n, _, r, c, v = P.csrc_to_triplets(a)
    assert r[0] == 0 and c[0] == 0 and v[0] == a.ad[0]
    d = O.build_csrc(n, r, c, v)
    for k in ("ad", "ia", "ja", "al", "au"):
        assert np.array_equal(d[k], getattr(a, k))
