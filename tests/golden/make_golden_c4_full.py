"""C4 at full scale (BASELINE configs[3]) pinned to the REFERENCE (this container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_c4_full.py [--ds-pairs 0,99] [--procs 6]

Model: the interlocking-course knit tube, 200 courses x 100,000 segments,
W = 100 stitches (~2e7 vertices).  Built here from the
course formula with numpy only (the same expression as
paper_2106_12655_b200.generators.knit_course; a per-course sha256 of the
vertex bytes is stored so the GPU test proves it rebuilt the same input).

What the reference computes:
* ``potential_link_search`` over the full model (pls.py:59-73)  -> the pair list;
* ``discretize`` over the full model (discretize.py:112-191)    -> vertex hashes
  (the knit tube needs no refinement; we record that the reference agrees);
* ``link_count_crossings`` (crossings.py:259-299) on ALL PLS pairs -> the integer
  linking numbers (the reference's own CC path, 0.9 s per pair);
* ``link_direct`` (direct.py:149-162, ``_link_atan``) on the sampled pairs
  given by --ds-pairs (1e10 segment pairs each, ~400 s each on one core)
  -> raw sums the CUDA path must match within 1e-9.

Writes tests/golden/golden_c4_full.json and prints a log (committed under
profiles/r02/).
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

COURSES, N, W = 200, 100_000, 100


def course(k, n=N, w=W, h=1.0, A=0.9, B=0.3):
    R = w * 1.5 / (2.0 * math.pi)
    s = 2.0 * math.pi * np.arange(n) / n
    sign = -1.0 if k % 2 else 1.0
    z = k * h + sign * A * np.sin(w * s)
    rho = R + sign * B * np.cos(w * s)
    return np.stack([rho * np.cos(s), rho * np.sin(s), z], axis=1)


def _cc(pair):
    import linkcert as ref
    i, j = pair
    t0 = time.perf_counter()
    v = ref.link_count_crossings(ref.PolylineLoop(course(i)), ref.PolylineLoop(course(j)))
    return i, j, int(v), time.perf_counter() - t0


def _ds(pair):
    import linkcert as ref
    i, j = pair
    t0 = time.perf_counter()
    v = ref.link_direct(ref.PolylineLoop(course(i)), ref.PolylineLoop(course(j)))
    return i, j, float(v), time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ds-pairs", default="0,99", help="comma list of k: sampled DS pairs (k, k+1)")
    ap.add_argument("--procs", type=int, default=6)
    args = ap.parse_args()
    import linkcert as ref

    ds_pairs = [(int(k), int(k) + 1) for k in args.ds_pairs.split(",") if k]
    ctx = mp.get_context("fork")
    pool = ctx.Pool(args.procs)
    # DS first: they are the long pole (one core each for ~400 s).
    ds_async = [pool.apply_async(_ds, (p,)) for p in ds_pairs]

    t0 = time.perf_counter()
    verts = [course(k) for k in range(COURSES)]
    hashes = [hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for v in verts]
    model = ref.CurveModel([ref.LoopGeometry.from_polyline(v) for v in verts])
    t_build = time.perf_counter() - t0
    print(f"reference model built in {t_build:.1f} s, xi = {model.xi!r}", flush=True)

    t0 = time.perf_counter()
    pairs = ref.potential_link_search(model)
    t_pls = time.perf_counter() - t0
    plist = [tuple(map(int, p)) for p in pairs]
    print(f"reference PLS: {len(plist)} pairs in {t_pls:.1f} s", flush=True)

    cc_async = pool.map_async(_cc, plist, chunksize=4)

    t0 = time.perf_counter()
    polys = ref.discretize(model, pairs)
    t_disc = time.perf_counter() - t0
    same = [hashlib.sha256(np.ascontiguousarray(p.vertices).tobytes()).hexdigest() == h
            for p, h in zip(polys, hashes)]
    print(f"reference discretize: {t_disc:.1f} s, vertices unchanged on {sum(same)}/{len(same)} loops",
          flush=True)
    del polys, model

    cc = cc_async.get()
    cc_time = sum(r[3] for r in cc)
    print(f"reference CC on {len(cc)} pairs: {cc_time:.1f} s of CPU time, values {sorted(set(r[2] for r in cc))}",
          flush=True)
    ds = [a.get() for a in ds_async]
    for i, j, v, t in ds:
        print(f"reference DS ({i},{j}): raw {v!r} in {t:.1f} s", flush=True)
    pool.close()
    pool.join()

    out = {
        "courses": COURSES, "n": N, "W": W,
        "course_sha256": hashes,
        "pls_pairs": [list(p) for p in plist],
        "discretize_unchanged": all(same),
        "cc": {f"{i},{j}": v for i, j, v, _ in sorted(cc)},
        "ds_raw": {f"{i},{j}": v for i, j, v, _ in ds},
        "reference_seconds": {"build": t_build, "pls": t_pls, "discretize": t_disc,
                              "cc_total_cpu": cc_time, "cc_per_pair_mean": cc_time / max(len(cc), 1),
                              "ds_per_pair": {f"{i},{j}": t for i, j, _, t in ds}},
    }
    (HERE / "golden_c4_full.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print("wrote golden_c4_full.json")


if __name__ == "__main__":
    main()
