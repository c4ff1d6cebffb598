"""Phase times of the moment-tree build (LC_BH_STATS=1) for one ribbon loop.

    python tools/bh_build_probe.py 1000000 4000000
"""
import os
import sys
import time

os.environ["LC_BH_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12655_b200 as lc  # noqa: E402
from paper_2106_12655_b200 import _native  # noqa: E402

ctx = _native.context()
for n in [int(x) for x in (sys.argv[1:] or ["1000000"])]:
    model, _ = lc.generators.double_helix_ribbon(10, n)
    a = model.loops[0].start_points()
    for rep in range(3):
        t0 = time.perf_counter()
        f = ctx.bh_forest(a, [0, n])
        t1 = time.perf_counter()
        tr = lc.build_moment_tree(a)
        t2 = time.perf_counter()
        print(f"n={n} rep={rep} forest {1e3 * (t1 - t0):.2f} ms, MomentTree {1e3 * (t2 - t1):.2f} ms",
              file=sys.stderr, flush=True)
        del f, tr
