"""Device CSRC construction (build_csr -> csr_to_csrc, csrc/assemble.cu) on the
BASELINE configs: triplets in csrc_to_csr order, shuffled with a fixed seed,
built on cuda:0 and compared bit for bit with the fixture; the reference's own
construction (oracle/_ref, one host core) timed beside it where it finishes in
reasonable time. Prints one JSON line per config."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1003_0952_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--ref-configs", default="c1,c2")
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    for cfg in args.configs.split(","):
        a, _, _ = P.config_matrix(cfg)
        n, _, r, c, v = P.csrc_to_triplets(a)
        perm = np.random.default_rng(1).permutation(r.size)
        r, c, v = r[perm], c[perm], v[perm]
        del perm
        best, phases = None, None
        for _ in range(args.reps):
            t = {}
            t0 = time.perf_counter()
            got = P.build_csrc((n, n, r, c, v), timings=t)
            dt = time.perf_counter() - t0
            if best is None or dt < best:
                best, phases = dt, t
        exact = (np.array_equal(got.ia, a.ia) and np.array_equal(got.ja, a.ja)
                 and np.array_equal(got.ad.view(np.int64), a.ad.view(np.int64))
                 and np.array_equal(got.al.view(np.int64), a.al.view(np.int64))
                 and np.array_equal(got.au.view(np.int64), a.au.view(np.int64)))
        line = dict(config=cfg, n=n, triplets=int(r.size), pairs=int(a.ja.size), gpu_s=best,
                    gpu_phases_ms=phases, bit_exact_vs_fixture=bool(exact),
                    triplets_per_s=r.size / best)
        if cfg in args.ref_configs.split(","):
            from oracle.oracle import Ref
            if Ref.available():
                t0 = time.perf_counter()
                ref = Ref().build_csrc(n, r, c, v)
                line["reference_cpu_s"] = time.perf_counter() - t0
                line["reference_cores"] = 1
                line["bit_exact_vs_reference"] = bool(
                    np.array_equal(ref["ja"], got.ja) and np.array_equal(ref["al"].view(np.int64), got.al.view(np.int64))
                    and np.array_equal(ref["au"].view(np.int64), got.au.view(np.int64)))
                line["speedup_vs_reference"] = line["reference_cpu_s"] / best
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
