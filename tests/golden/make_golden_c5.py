"""C5 accuracy/throughput sweep (BASELINE configs[4]) pinned to the REFERENCE (this container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_c5.py [--procs 2]

Two curve pairs with a known linking number, n segments per loop,
n in {1e3, 1e4, 1e5, 1e6}:
* ``ribbon``: ``generators.double_helix_ribbon(10, n)`` (generators.py:96-115), lambda = +10;
* ``yarn``: two adjacent courses of the knit tube (SURVEY Appendix B.3,
  W = 100 stitches), lambda = -100.

For each case the reference's three methods, timed on one core here:
* direct summation ``link_direct`` (direct.py:149-162): n <= 1e5 (n = 1e5 is
  1e10 segment pairs, ~400 s); n = 1e6 is not run (~11 h) and is marked
  extrapolated from the 1e5 time by n^2 (DS cost is exactly proportional);
* Barnes-Hut ``build_moment_tree`` + ``barnes_hut_detailed`` with default
  ``BarnesHutParams`` (barneshut.py:326,355-371);
* crossing counting ``link_count_crossings`` (crossings.py:259-299).

Writes tests/golden/golden_c5.json (values, errors vs the known lambda,
times, per-loop vertex sha256 so the GPU test proves it rebuilt the inputs).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

NS = (1_000, 10_000, 100_000, 1_000_000)
DS_MAX_N = 100_000


def yarn_course(k, n, w=100, h=1.0, A=0.9, B=0.3):
    R = w * 1.5 / (2.0 * math.pi)
    s = 2.0 * math.pi * np.arange(n) / n
    sign = -1.0 if k % 2 else 1.0
    z = k * h + sign * A * np.sin(w * s)
    rho = R + sign * B * np.cos(w * s)
    return np.stack([rho * np.cos(s), rho * np.sin(s), z], axis=1)


def case_loops(name, n):
    import linkcert as ref
    if name == "ribbon":
        from linkcert import generators as rg
        model, _ = rg.double_helix_ribbon(10, n)
        return [lp.control_points for lp in model.loops], 10
    if name == "yarn":
        return [yarn_course(0, n), yarn_course(1, n)], -100
    raise KeyError(name)


def _ds(job):
    import linkcert as ref
    name, n = job
    (a, b), _ = case_loops(name, n)
    t0 = time.perf_counter()
    v = ref.link_direct(ref.PolylineLoop(a), ref.PolylineLoop(b))
    return name, n, float(v), time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=2)
    args = ap.parse_args()
    import linkcert as ref

    # warm the numba JIT once so no timing includes compilation
    (a, b), _ = case_loops("ribbon", 200)
    pa, pb = ref.PolylineLoop(a), ref.PolylineLoop(b)
    ref.link_direct(pa, pb)
    ref.barnes_hut_detailed(ref.build_moment_tree(pa), ref.build_moment_tree(pb))
    ref.link_count_crossings(pa, pb)

    pool = mp.get_context("fork").Pool(args.procs)
    big = [pool.apply_async(_ds, ((name, DS_MAX_N),)) for name in ("ribbon", "yarn")]
    out = {}
    for name in ("ribbon", "yarn"):
        for n in NS:
            (a, b), lam = case_loops(name, n)
            pa, pb = ref.PolylineLoop(a), ref.PolylineLoop(b)
            rec = {"n": n, "lambda": lam,
                   "sha256": [hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for v in (a, b)]}
            if n < DS_MAX_N:
                t0 = time.perf_counter()
                rec["ds_raw"] = float(ref.link_direct(pa, pb))
                rec["ds_seconds"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            t1_, t2_ = ref.build_moment_tree(pa), ref.build_moment_tree(pb)
            t1 = time.perf_counter()
            bh = ref.barnes_hut_detailed(t1_, t2_)
            t2 = time.perf_counter()
            rec.update(bh_value=bh.value, bh_beta_used=bh.beta_used, bh_reran=bh.reran,
                       bh_e_estimate=bh.e_estimate, bh_build_seconds=t1 - t0, bh_eval_seconds=t2 - t1)
            del t1_, t2_
            t0 = time.perf_counter()
            try:
                rec["cc_value"] = int(ref.link_count_crossings(pa, pb))
            except Exception as e:  # noqa: BLE001 - recorded, not hidden
                rec["cc_error"] = f"{type(e).__name__}: {e}"
            rec["cc_seconds"] = time.perf_counter() - t0
            out[f"{name}/{n}"] = rec
            print(json.dumps({"case": f"{name}/{n}", **{k: v for k, v in rec.items() if k != "sha256"}}), flush=True)
    for r in big:
        name, n, v, t = r.get()
        out[f"{name}/{n}"].update(ds_raw=v, ds_seconds=t)
        print(json.dumps({"case": f"{name}/{n}", "ds_raw": v, "ds_seconds": t}), flush=True)
    for name in ("ribbon", "yarn"):
        t5 = out[f"{name}/{DS_MAX_N}"]["ds_seconds"]
        out[f"{name}/1000000"]["ds_seconds_extrapolated"] = t5 * (1_000_000 / DS_MAX_N) ** 2
    pool.close()
    pool.join()
    (HERE / "golden_c5.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print("wrote golden_c5.json")


if __name__ == "__main__":
    main()
