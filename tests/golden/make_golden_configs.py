"""Config-scale golden data from the REFERENCE ITSELF (oracle/_ref, compiled
from /root/reference): pins the product's plan functions, colourings, device
construction and the oracle's y at BASELINE sizes (C1-C5), where committing
the arrays themselves would be too large. Runs here only (the reference tree
is absent on the GPU box); the outputs travel with the repo.

  configs.json
    partitions[cfg][p]   partition_by_nnz block_start / block_nnz, effective_ranges
                         lo / hi, build_interval_plan boundaries + intervals
                         (partition.hpp:55-134), p in {2, 3, 4, 8, 16, 148}
    y_sha256[cfg]        sha256 of the reference's sequential spmv_csrc y
                         (kernels.hpp:25-43) on the config's x, and of its
                         spmv_csrc_transpose (kernels.hpp:47-65)
    construction[cfg]    the reference's build_csr -> csr_to_csrc (csr.hpp:55-92,
                         csrc_matrix.hpp:44-91) of the fixture's triplets in a
                         seeded shuffled order: sha256 of ad / ia / ja / al / au
                         (asserted equal to the fixture here)
    colorings[cfg][mode/order]  n_colors, class sizes, edge counts, sha256 of the
                         reference's color_rows(build_conflict_graph) colours
                         (coloring.hpp:93-164) -- C1 and C2
    colour_validity[cfg] the product's scalable colouring (csrc_color_rows,
                         neighbourhood / natural) at C3-C5 checked by the
                         reference's validate_coloring (coloring.hpp:175-198):
                         its sha256, n_colors, and the reference's verdict
  colorings_c1c2.npz     the reference's colours themselves at C1 / C2

Usage: python tests/golden/make_golden_configs.py [c1,c2,...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Ref, config_fixture  # noqa: E402

PS = [2, 3, 4, 8, 16, 148]
SHUFFLE_SEED = 2026
COLOR_CASES = [("neighborhood", 0, "natural", 0), ("exact", 1, "natural", 0),
               ("neighborhood", 0, "largest_first", 1), ("exact", 1, "largest_first", 1)]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fixture_triplets(a):
    """csrc_to_csr order (csrc_matrix.hpp:95-108): per row (i,i,ad), then per
    stored pair (i,j,al), (j,i,au); numpy, no product code."""
    n = a.n
    cnt = np.diff(a.ia.astype(np.int64))
    rows_of = np.repeat(np.arange(n, dtype=np.int32), cnt)
    per_row = 1 + 2 * cnt
    start = np.concatenate([[0], np.cumsum(per_row)[:-1]]).astype(np.int64)
    m = int(per_row.sum())
    r = np.empty(m, np.int32)
    c = np.empty(m, np.int32)
    v = np.empty(m, np.float64)
    r[start] = np.arange(n, dtype=np.int32)
    c[start] = np.arange(n, dtype=np.int32)
    v[start] = a.ad
    t = np.arange(a.ja.size, dtype=np.int64)
    base = start[rows_of] + 1 + 2 * (t - a.ia[rows_of].astype(np.int64))
    r[base], c[base], v[base] = rows_of, a.ja, a.al
    r[base + 1], c[base + 1], v[base + 1] = a.ja, rows_of, a.au
    return r, c, v


def shuffled_triplets(a):
    r, c, v = fixture_triplets(a)
    perm = np.random.default_rng(SHUFFLE_SEED).permutation(r.size)
    return r[perm], c[perm], v[perm]


def main():
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4", "c5"]
    only_y = len(sys.argv) > 2 and sys.argv[2] == "--only-y"  # refresh the y hashes alone
    out_path = os.path.join(HERE, "configs.json")
    out = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for key in ("partitions", "y_sha256", "construction", "colorings", "colour_validity"):
        out.setdefault(key, {})
    out["shuffle_seed"] = SHUFFLE_SEED
    R = Ref()  # the x86-64-v2 build: no FMA contraction (oracle/oracle.py)
    npz = {}
    npz_path = os.path.join(HERE, "colorings_c1c2.npz")
    if os.path.exists(npz_path):
        z = np.load(npz_path)
        npz = {k: z[k] for k in z.files}
    for cfg in cfgs:
        t0 = time.time()
        a, x = config_fixture(cfg)
        print(f"{cfg}: n={a.n} k={a.k_off()} fixture {time.time() - t0:.1f}s", flush=True)
        parts = {}
        for p in PS:
            bs, bn = R.partition_by_nnz(a, p)
            lo, hi = R.effective_ranges(a, bs)
            bd, ivs = R.interval_plan(lo, hi)
            parts[str(p)] = dict(block_start=bs, block_nnz=bn, lo=lo, hi=hi, boundaries=bd,
                                 intervals=[[b, e, c] for b, e, c in ivs])
        out["partitions"][cfg] = parts
        y = R.spmv_csrc(a, x)
        yt = R.spmv_csrc(a, x, transpose=True)
        out["y_sha256"][cfg] = dict(y=sha(y), yt=sha(yt), y_norm=float(np.linalg.norm(y)))
        print(f"  partitions + y {time.time() - t0:.1f}s", flush=True)
        if only_y:
            with open(out_path, "w") as f:
                json.dump(out, f, separators=(",", ":"))
            continue
        if cfg in ("c3", "c5"):
            r, c, v = shuffled_triplets(a)
            b = R.build_csrc(a.n, r, c, v)
            del r, c, v
            for f in ("ad", "ia", "ja", "al", "au"):
                assert np.array_equal(b[f], getattr(a, f)), (cfg, f)
            out["construction"][cfg] = dict(
                triplets=int(a.n + 2 * a.k_off()), value_symmetric=bool(b["value_symmetric"]),
                **{f: sha(b[f]) for f in ("ad", "ia", "ja", "al", "au")})
            del b
            print(f"  construction {time.time() - t0:.1f}s", flush=True)
        if cfg in ("c1", "c2"):
            cols = {}
            for mname, mode, oname, order in COLOR_CASES:
                color, nc, (nd, ni) = R.color_rows(a, mode, order)
                sizes = np.bincount(color, minlength=nc).tolist()
                cols[f"{mname}/{oname}"] = dict(n_colors=nc, class_sizes=sizes, n_direct=nd, n_indirect=ni,
                                                sha256=sha(color.astype(np.int32)))
                if order == 0:
                    npz[f"{cfg}_{mname}"] = color.astype(np.uint8)
                print(f"  colour {mname}/{oname}: {nc} colours {time.time() - t0:.1f}s", flush=True)
            out["colorings"][cfg] = cols
        else:
            import paper_1003_0952_b200 as P  # the product colouring under test, validated by the reference
            pa = P.CsrcMatrix(a.n, a.ad, a.ia, a.ja, a.al, a.au)
            col = P.color_rows(pa, P.ConflictMode.neighborhood, P.ColorOrder.natural)
            ok, ra, rb, q = R.validate_coloring(a, col.color, col.n_colors)
            assert ok, (cfg, ra, rb, q)
            out["colour_validity"][cfg] = dict(mode="neighborhood", order="natural", n_colors=col.n_colors,
                                               sha256=sha(col.color.astype(np.int32)), reference_valid=ok,
                                               class_sizes=np.bincount(col.color, minlength=col.n_colors).tolist())
            print(f"  product colouring validated by the reference {time.time() - t0:.1f}s", flush=True)
        with open(out_path, "w") as f:
            json.dump(out, f, separators=(",", ":"))
        np.savez_compressed(npz_path, **npz)
    print("wrote", out_path, npz_path)


if __name__ == "__main__":
    main()
