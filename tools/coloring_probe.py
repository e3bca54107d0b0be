"""Host coloring at config scale: color_rows time, colour
count and validate_coloring for neighbourhood / exact modes (natural order)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1003_0952_b200 as P  # noqa: E402

for name in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2"]):
    t = time.time()
    a, x, _ = P.config_matrix(name)
    tg = time.time() - t
    for mode in (P.ConflictMode.neighborhood, P.ConflictMode.exact):
        t = time.time()
        c = P.color_rows(a, mode)
        tc = time.time() - t
        t = time.time()
        v = P.validate_coloring(a, c)
        tv = time.time() - t
        print(f"{name} n={a.n} gen {tg:.1f}s {mode.name:12s} colors {c.n_colors:3d} color_rows {tc:7.2f}s "
              f"validate {tv:5.2f}s valid={v.valid}", flush=True)
