"""The product's host planners (paper_1003_0952_b200/csrc/plan_host.cpp) are
bit-exact with the reference's scheduling layer (partition.hpp, coloring.hpp,
parallel.hpp ColorfulPlan::slice): checked against golden vectors produced by
the reference itself and against the reference's known answers."""
import numpy as np
import pytest

import paper_1003_0952_b200 as P

from .helpers import family, known_answers, matrix_from_dict

KA = known_answers()
FAM = family()


def test_partition_known_answer():
    ka = KA["partition_counts"]
    part = P.partition_by_nnz(matrix_from_dict(ka["matrix"]), ka["p"])
    assert part.block_start == ka["block_start"] and part.block_nnz == ka["block_nnz"]


def test_partition_errors_like_the_reference():
    a = matrix_from_dict(KA["tridiag4_coloring"]["matrix"])
    with pytest.raises(P.Error, match=r"need 1 <= p <= n, got p=5, n=4"):
        P.partition_by_nnz(a, 5)
    with pytest.raises(P.Error, match=r"got p=0"):
        P.partition_by_nnz(a, 0)


def test_effective_ranges_known_answers():
    for case in KA["effective_ranges"]["cases"]:
        a = matrix_from_dict(case["matrix"])
        bs = case["block_start"]
        part = P.RowPartition(len(bs) - 1, bs, [0] * (len(bs) - 1))
        r = P.effective_ranges(a, part)
        assert [e.lo for e in r] == case["lo"] and [e.hi for e in r] == case["hi"]


def test_interval_plan_known_answers():
    for case in KA["interval_plans"]["cases"]:
        ip = P.build_interval_plan([P.EffectiveRange(l, h) for l, h in zip(case["lo"], case["hi"])])
        assert ip.boundaries == case["boundaries"]
        assert [[b, e, c] for b, e, c in ip.intervals] == [[b, e, c] for b, e, c in case["intervals"]]


def test_coloring_known_answers():
    ka = KA["tridiag4_coloring"]
    a = matrix_from_dict(ka["matrix"])
    for mode, key in ((P.ConflictMode.neighborhood, "neighborhood"), (P.ConflictMode.exact, "exact")):
        c = P.color_rows(a, mode)
        assert c.color.tolist() == ka[key]["color"] and c.n_colors == ka[key]["n_colors"]
        assert list(P.conflict_edge_counts(a, mode)) == ka[key]["edges"]


def test_validate_coloring_reports_first_violation():
    a = matrix_from_dict(KA["tridiag4_coloring"]["matrix"])
    v = P.validate_coloring(a, P.Coloring(np.array([0, 0, 1, 1], np.int32), 2))
    assert (v.valid, v.row_a, v.row_b, v.position) == (False, 0, 1, 0)
    # singleton classes are always valid (test_coloring.cpp:152-159)
    assert P.validate_coloring(a, P.Coloring(np.arange(4, dtype=np.int32), 4)).valid


def test_edgeless_graph_needs_one_color():
    a = P.CsrcMatrix(6, np.ones(6), np.zeros(7, np.int32), [], [], [])
    c = P.color_rows(a)
    assert c.n_colors == 1 and c.classes[0].size == 6


@pytest.mark.parametrize("idx", range(29))
def test_family_partitions_ranges_intervals(idx):
    p = f"m{idx}_"
    a = FAM.matrix(p)
    for pp in (1, 2, 3, 4, 8):
        if not FAM.has(p + f"p{pp}_bs"):
            continue
        part = P.partition_by_nnz(a, pp)
        assert part.block_start == FAM[p + f"p{pp}_bs"].tolist()
        assert part.block_nnz == FAM[p + f"p{pp}_bn"].tolist()
        r = P.effective_ranges(a, part)
        assert [e.lo for e in r] == FAM[p + f"p{pp}_lo"].tolist()
        assert [e.hi for e in r] == FAM[p + f"p{pp}_hi"].tolist()
        ip = P.build_interval_plan(r)
        assert ip.boundaries == FAM[p + f"p{pp}_bd"].tolist()
        assert [[b, e] for b, e, _ in ip.intervals] == FAM[p + f"p{pp}_iv"].tolist()
        flat = [m for _, _, c in ip.intervals for m in c]
        assert flat == FAM[p + f"p{pp}_ivm"].tolist()


@pytest.mark.parametrize("idx", range(29))
def test_family_colorings_all_modes_and_orders(idx):
    p = f"m{idx}_"
    if not FAM.has(p + "col00"):
        pytest.skip("no colouring stored")
    a = FAM.matrix(p)
    for mode in (0, 1):
        assert list(P.conflict_edge_counts(a, P.ConflictMode(mode))) == FAM[p + f"edges{mode}"].tolist()
        for order in (0, 1, 2):
            c = P.color_rows(a, P.ConflictMode(mode), P.ColorOrder(order))
            assert c.color.tolist() == FAM[p + f"col{mode}{order}"].tolist()
            assert c.n_colors == int(FAM[p + f"nc{mode}{order}"])
            assert P.validate_coloring(a, c).valid


@pytest.mark.parametrize("idx", range(29))
def test_family_colorful_slices(idx):
    p = f"m{idx}_"
    if not FAM.has(p + "slices4"):
        pytest.skip("no slices stored")
    a = FAM.matrix(p)
    plan = P.ColorfulPlan(P.color_rows(a))
    plan.slice(a, 4)
    assert np.array_equal(plan.class_slices, FAM[p + "slices4"])


def test_local_buffers_plan_build():
    a = FAM.matrix("m0_")
    lb = P.LocalBuffersPlan.build(a, 3)
    assert lb.partition.block_start == FAM["m0_p3_bs"].tolist()


def test_allocation_stats():
    S = P.Strategy
    assert P.allocation_stats(S(P.StrategyKind.local_buffers, p=4)) == 4
    assert P.allocation_stats(S(P.StrategyKind.local_buffers, p=1)) == 0
    assert P.allocation_stats(S(P.StrategyKind.colorful, p=4)) == 0


def test_working_set_kb_known_answers():
    for n, nnz, vs, kb in KA["working_set_kb"]["rows"]:
        assert int(P.working_set_kb(n, nnz, vs)) == kb
    with pytest.raises(P.Error):
        P.working_set_kb(0, 0, False)
