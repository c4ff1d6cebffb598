"""Barnes-Hut vs direct summation on the GPU for one yarn-like loop pair
(double_helix_ribbon(10, n)).

    python tools/bh_probe.py [--sizes 10000 100000 1000000] [--ds-max 1000000]

Prints one JSON line per size: tree build ms (both loops), traversal ms,
node pairs visited, value / error vs the exact linking number, and the direct
summation time for the same pair.  Wall-clock around synchronous library calls
(each returns after its own stream sync), best of 3.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2106_12655_b200 as lc  # noqa: E402
from paper_2106_12655_b200 import _native  # noqa: E402


def best(fn, reps=3):
    out, t = None, float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        t = min(t, time.perf_counter() - t0)
    return out, t * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", type=int, nargs="+", default=[10_000, 100_000, 1_000_000])
    ap.add_argument("--ds-max", type=int, default=1_000_000)
    ap.add_argument("--lam", type=int, default=10)
    ap.add_argument("--kusari", action="store_true", help="also: the C3 tube certificate with the bh kernel")
    args = ap.parse_args()
    ctx = _native.context()
    if args.kusari:
        import numpy as np
        from paper_2106_12655_b200 import barneshut

        model = lc.generators.kusari_tube()
        pairs = np.array(list(lc.potential_link_search(model)), dtype=np.int64)
        polys = lc.discretize(model, lc.potential_link_search(model))
        (val, est, beta, reran), ms = best(lambda: barneshut.evaluate_pairs(polys, pairs))
        ds = lc.compute_linking_matrix(model)
        lk = np.rint(val).astype(np.int64)
        want = {(i, j): v for i, j, v in ds.entries}
        agree = all(want.get((int(i), int(j)), 0) == int(v) for (i, j), v in zip(pairs, lk))
        t = {}
        _, cert_ms = best(lambda: lc.compute_linking_matrix(model, choice=lc.KernelChoice(method="bh"), timings=t))
        print(json.dumps({"kusari_pairs": len(pairs), "bh_batched_ms": round(ms, 3), "reran": int(reran.sum()),
                          "max_err": float(np.max(np.abs(val - lk))), "agrees_with_ds": agree,
                          "bh_certificate_ms": round(cert_ms, 3), "timings": t}), flush=True)
    for n in args.sizes:
        model, _ = lc.generators.double_helix_ribbon(args.lam, n)
        a, b = (lp.start_points() for lp in model.loops)
        lc.barnes_hut_detailed(lc.build_moment_tree(a[:64]), lc.build_moment_tree(b[:64]))   # warm
        (ta, tb), build_ms = best(lambda: (lc.build_moment_tree(a), lc.build_moment_tree(b)))
        res, total_ms = best(lambda: lc.barnes_hut_detailed(ta, tb))
        _, _, visits = ta._forest.eval(tb._forest, [[0, 0]], res.beta_used)
        _, one_ms = best(lambda: ta._forest.eval(tb._forest, [[0, 0]], 2.0))
        line = {"n": n, "seg_pairs": n * n, "bh_build_ms": round(build_ms, 3), "bh_eval_ms": round(total_ms, 3),
                "bh_single_traversal_ms": round(one_ms, 3), "visits_at_beta_used": visits,
                "value": res.value, "err": abs(res.value - args.lam), "beta_used": res.beta_used,
                "reran": res.reran, "e_estimate": res.e_estimate}
        if n <= args.ds_max:
            raw, ds_ms = best(lambda: ctx.link_direct(a, b), reps=2)
            line.update(ds_ms=round(ds_ms, 3), ds_value=float(raw), ds_rate=n * n / (ds_ms * 1e-3))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
