"""Device CSRC construction (csrc/assemble.cu) against the compiled reference
(oracle/_ref: build_csr csr.hpp:55-92, csr_to_csrc csrc_matrix.hpp:44-91,
decompose_rect csrc_matrix.hpp:113-142) and the golden fixtures.

Bar: bit-exact (ad, ia, ja, al, au, value_symmetric; CSR row_ptr, col_idx,
values) and the reference's error messages. Duplicates: the reference sums a
run of equal (row, col) in its std::sort order, which is unspecified for runs
of three or more (introsort is not stable); the device sums them in input
order. Runs of two are exact (a + b == b + a); longer runs are checked against
the reference to within (run length - 1) * eps * sum|v|, and bit-exactly
against an input-order sum."""
import numpy as np
import pytest

import paper_1003_0952_b200 as P
from oracle.oracle import Oracle, Ref
from tests.helpers import known_answers, matrix_from_dict, meshes, family

pytestmark = pytest.mark.gpu
KA = known_answers()


def same_bits(a, b):
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.int64), b.view(np.int64))


def assert_csrc_equal(got, ref):
    assert got.n == ref["n"]
    assert np.array_equal(got.ia, ref["ia"])
    assert np.array_equal(got.ja, ref["ja"])
    assert same_bits(got.ad, ref["ad"])
    assert same_bits(got.al, ref["al"])
    assert got.value_symmetric == ref["value_symmetric"]
    if not got.value_symmetric:
        assert same_bits(got.au, ref["au"])
    else:
        assert got.au.size == 0


def csrc_dict(a):
    return dict(n=a.n, ad=a.ad, ia=a.ia, ja=a.ja, al=a.al, au=a.au if not a.value_symmetric else np.zeros(0),
                value_symmetric=a.value_symmetric)


def test_pair_placement_known_answer():
    """test_core.cpp:147-161: tridiagonal-ish pairs land at (row, lower col)."""
    want = matrix_from_dict(KA["pair_placement"]["matrix"])
    n, _, r, c, v = P.csrc_to_triplets(want)
    got = P.build_csrc((n, n, r[::-1].copy(), c[::-1].copy(), v[::-1].copy()))
    assert_csrc_equal(got, csrc_dict(want))


@pytest.mark.parametrize("g", range(4))
def test_mesh_round_trip_bit_exact(g):
    """csrc -> triplets (csrc_to_csr order) -> device build == the reference-built
    golden mesh CSRC (test_core.cpp:173-194 round trip), also from shuffled input."""
    a = meshes().matrix(f"g{g}_")
    n, _, r, c, v = P.csrc_to_triplets(a)
    assert_csrc_equal(P.build_csrc((n, n, r, c, v)), csrc_dict(a))
    perm = np.random.default_rng(g).permutation(r.size)
    assert_csrc_equal(P.build_csrc((n, n, r[perm], c[perm], v[perm])), csrc_dict(a))


@pytest.mark.parametrize("idx", range(0, 29, 4))
def test_family_triplets_match_reference(idx):
    """The reference's own generator families: triplets -> CSRC on the device
    and through the compiled reference, bit for bit."""
    fam = family()
    a = fam.matrix(f"m{idx}_")
    n, _, r, c, v = P.csrc_to_triplets(a)
    perm = np.random.default_rng(100 + idx).permutation(r.size)
    r, c, v = r[perm], c[perm], v[perm]
    ref = Ref().build_csrc(n, r, c, v)
    assert_csrc_equal(P.build_csrc((n, n, r, c, v)), ref)


@pytest.mark.parametrize("seed", range(6))
def test_reference_generators_bit_exact(seed):
    R = Ref()
    for vs in (False, True):
        r, c, v = R.gen_random_sym(40 + 17 * seed, 0.08 + 0.03 * seed, 1000 + seed, vs)
        n = 40 + 17 * seed
        ref = R.build_csrc(n, r, c, v)
        got = P.build_csrc((n, n, r, c, v))
        assert_csrc_equal(got, ref)
        assert got.value_symmetric == vs


def _dups(seed, n, m, max_run):
    rng = np.random.default_rng(seed)
    # symmetric pattern with a diagonal; every pair emitted 1..max_run times per side
    rows, cols = [], []
    for i in range(n):
        rows.append(i)
        cols.append(i)
        for j in rng.choice(i, size=min(i, 3), replace=False) if i else []:
            rows += [i, int(j)]
            cols += [int(j), i]
    base_r, base_c = np.array(rows, np.int32), np.array(cols, np.int32)
    reps = rng.integers(1, max_run + 1, base_r.size)
    r = np.repeat(base_r, reps)
    c = np.repeat(base_c, reps)
    v = rng.standard_normal(r.size) * 10.0 ** rng.uniform(-3, 3, r.size)
    perm = rng.permutation(r.size)
    return r[perm], c[perm], v[perm]


@pytest.mark.parametrize("seed", range(4))
def test_duplicate_pairs_bit_exact(seed):
    """Runs of at most two duplicates: exact whatever the sort order."""
    n = 50 + 10 * seed
    r, c, v = _dups(seed, n, 0, 2)
    ref = Ref().build_csrc(n, r, c, v)
    assert_csrc_equal(P.build_csrc((n, n, r, c, v)), ref)
    rp, ci, va = Ref().build_csr(n, n, r, c, v)
    csr = P.build_csr((n, n, r, c, v))
    assert np.array_equal(csr.row_ptr, rp) and np.array_equal(csr.col_idx, ci) and same_bits(csr.values, va)


@pytest.mark.parametrize("seed", range(3))
def test_long_duplicate_runs(seed):
    """Runs of up to 8 duplicates: bit-exact with an input-order sum, and within
    (run - 1) eps sum|v| of the reference's (unspecified-order) sum."""
    n = 40
    r, c, v = _dups(seed, n, 0, 8)
    csr = P.build_csr((n, n, r, c, v))
    rp, ci, va = Ref().build_csr(n, n, r, c, v)
    assert np.array_equal(csr.row_ptr, rp) and np.array_equal(csr.col_idx, ci)
    key = r.astype(np.int64) * n + c
    order = np.argsort(key, kind="stable")
    ks = key[order]
    heads = np.flatnonzero(np.r_[True, ks[1:] != ks[:-1]])
    ends = np.r_[heads[1:], ks.size]
    want = np.empty(heads.size)
    bound = np.empty(heads.size)
    for q, (b, e) in enumerate(zip(heads, ends)):
        s = v[order[b]]
        for t in range(b + 1, e):
            s = s + v[order[t]]
        want[q] = s
        bound[q] = (e - b) * np.finfo(np.float64).eps * np.abs(v[order[b:e]]).sum()
    assert same_bits(csr.values, want)
    assert np.all(np.abs(csr.values - va) <= bound)


def test_empty_and_diagonal_only():
    got = P.build_csrc((3, 3, [2, 0, 1], [2, 0, 1], [3.0, 1.0, 2.0]))
    assert got.ia.tolist() == [0, 0, 0, 0] and got.ad.tolist() == [1.0, 2.0, 3.0]
    assert got.value_symmetric  # no pairs: every pair matches (csrc_matrix.hpp:84-88)
    csr = P.build_csr((4, 2, [], [], []))
    assert csr.row_ptr.tolist() == [0, 0, 0, 0, 0] and csr.nnz() == 0


def test_errors_match_reference_wording():
    R = Ref()
    cases = [
        (3, [0, 1, 5, 2], [0, 1, 0, 7], [1.0] * 4),                # first out-of-bounds: (5, 0)
        (3, [0, 1, 2, 2], [0, 1, 2, 0], [1.0] * 4),                # (2, 0) has no transpose
        (3, [0, 1, 2, 0], [0, 1, 2, 2], [1.0] * 4),                # (0, 2) has no transpose (upper)
        (3, [0, 2, 1, 0, 2], [0, 2, 0, 1, 1], [1.0] * 5),          # row 1 lacks a diagonal, after its entries
        (4, [0, 1, 1, 3], [0, 1, 1, 3], [1.0] * 4),                # row 2 empty: no diagonal
        (3, [0, 1, 1, 2, 2, 1], [0, 1, 2, 1, 0, 1], [1.0] * 6),    # (2,0) missing vs row 1 ok
    ]
    for n, r, c, v in cases:
        with pytest.raises(ValueError) as ref_err:
            R.build_csrc(n, r, c, v)
        with pytest.raises(P.Error) as got_err:
            P.build_csrc((n, n, r, c, v))
        assert str(got_err.value) == str(ref_err.value)
    with pytest.raises(P.Error, match="csr_to_csrc: matrix is not square"):
        P.csr_to_csrc(P.CsrMatrix(2, 3, np.array([0, 0, 0]), np.zeros(0), np.zeros(0)))


def test_csr_to_csrc_entry_point():
    a = meshes().matrix("g0_")
    n, _, r, c, v = P.csrc_to_triplets(a)
    rp, ci, va = Ref().build_csr(n, n, r, c, v)
    got = P.csr_to_csrc(P.CsrMatrix(n, n, rp, ci, va))
    assert_csrc_equal(got, csrc_dict(a))


def test_decompose_rect_matches_reference():
    rng = np.random.default_rng(5)
    a = meshes().matrix("g0_")
    n, _, r, c, v = P.csrc_to_triplets(a)
    extra = 37
    tr = rng.integers(0, n, 600).astype(np.int32)
    tc = (n + rng.integers(0, extra, 600)).astype(np.int32)
    tv = rng.standard_normal(600)
    R = Ref()
    rp, ci, va = R.build_csr(n, n + extra, np.r_[r, tr], np.r_[c, tc], np.r_[v, tv])
    sq_ref, (trp, tci, tva) = R.decompose_rect(n, n + extra, rp, ci, va)
    got = P.decompose_rect(P.CsrMatrix(n, n + extra, rp, ci, va))
    assert_csrc_equal(got.square, sq_ref)
    assert got.m == n + extra
    assert np.array_equal(got.rect.row_ptr, trp) and np.array_equal(got.rect.col_idx, tci)
    assert same_bits(got.rect.values, tva)
    with pytest.raises(P.Error, match=r"decompose_rect: requires n_cols > n_rows \(got 3x3\)"):
        P.decompose_rect(P.CsrMatrix(3, 3, np.zeros(4, np.int32), np.zeros(0), np.zeros(0)))


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_config_round_trip(cfg):
    """BASELINE C1/C2 fixtures: triplets in csrc_to_csr order, shuffled, rebuilt
    on the device, bit-identical to the fixture (pinned to the reference in
    tests/test_fixtures.py); and to the reference's own build of the same triplets."""
    a, _, _ = P.config_matrix(cfg)
    n, _, r, c, v = P.csrc_to_triplets(a)
    perm = np.random.default_rng(7).permutation(r.size)
    r, c, v = r[perm], c[perm], v[perm]
    got = P.build_csrc((n, n, r, c, v))
    assert_csrc_equal(got, csrc_dict(a))
    if cfg == "c1":
        assert_csrc_equal(got, Ref().build_csrc(n, r, c, v))
