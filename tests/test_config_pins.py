"""Config-scale pins against the reference itself (tests/golden/configs.json,
made by tests/golden/make_golden_configs.py from oracle/_ref): the product's
host plan functions and colourings, and the oracle's y, at the BASELINE
configs C1-C5 -- not only on the <= 300-row golden family.

  * partition_by_nnz / effective_ranges / build_interval_plan
    (partition.hpp:55-134) for p in {2, 3, 4, 8, 16, 148}: bit-exact;
  * color_rows(build_conflict_graph) (coloring.hpp:93-164) at C1 / C2 in both
    conflict modes, natural and largest_first order: identical colours;
  * at C3-C5 (where the reference's std::set graph does not fit) the product's
    colouring is the one the reference's validate_coloring accepted;
  * the oracle's spmv_csrc / spmv_csrc_transpose y hash equal the reference's
    at full size, so the GPU parity tests' checker is itself pinned there.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from oracle.oracle import Oracle

import paper_1003_0952_b200 as P

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
with open(os.path.join(GOLDEN, "configs.json")) as _f:
    G = json.load(_f)
COLORS = np.load(os.path.join(GOLDEN, "colorings_c1c2.npz"))
O = Oracle()


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CFGS = ["c1", "c2", "c3", "c4", "c5"]


def check_partitions(cfg, a):
    for p, g in G["partitions"][cfg].items():
        part = P.partition_by_nnz(a, int(p))
        assert part.block_start == g["block_start"], p
        assert part.block_nnz == g["block_nnz"], p
        rng = P.effective_ranges(a, part)
        assert [r.lo for r in rng] == g["lo"] and [r.hi for r in rng] == g["hi"], p
        ip = P.build_interval_plan(rng)
        assert ip.boundaries == g["boundaries"], p
        assert [[b, e, c] for b, e, c in ip.intervals] == g["intervals"], p


def check_oracle_y(cfg, a, x):
    g = G["y_sha256"][cfg]
    assert sha(O.spmv_csrc(a, x)) == g["y"]
    assert sha(O.spmv_csrc(a, x, transpose=True)) == g["yt"]


def check_colorings(cfg, a):
    for case, g in G["colorings"][cfg].items():
        mode, order = case.split("/")
        col = P.color_rows(a, P.ConflictMode[mode], P.ColorOrder[order])
        assert col.n_colors == g["n_colors"], case
        assert sha(col.color.astype(np.int32)) == g["sha256"], case
        assert np.bincount(col.color, minlength=col.n_colors).tolist() == g["class_sizes"], case
        if order == "natural":
            assert np.array_equal(col.color, COLORS[f"{cfg}_{mode}"].astype(np.int32)), case
        assert P.conflict_edge_counts(a, P.ConflictMode[mode]) == (g["n_direct"], g["n_indirect"]), case


def check_validated_coloring(cfg, a):
    g = G["colour_validity"][cfg]
    assert g["reference_valid"]
    col = P.color_rows(a, P.ConflictMode.neighborhood, P.ColorOrder.natural)
    assert col.n_colors == g["n_colors"]
    assert sha(col.color.astype(np.int32)) == g["sha256"]
    assert P.validate_coloring(a, col).valid


@pytest.mark.parametrize("cfg", CFGS)
def test_config_pins(cfg):
    """One fixture build per config: partition maps (p in {2,3,4,8,16,148}),
    the oracle's y / y^T, and the colourings (C1/C2: equal to the reference's;
    C3-C5: the product colouring the reference's validate_coloring accepted)."""
    a, x, _ = P.config_matrix(cfg)
    check_partitions(cfg, a)
    check_oracle_y(cfg, a, x)
    if cfg in G["colorings"]:
        check_colorings(cfg, a)
    else:
        check_validated_coloring(cfg, a)
