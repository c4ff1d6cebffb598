"""Randomized certificate parity sweep, CUDA path vs the CPU oracle (GPU box).

    python tools/fuzz_parity.py --cases 200 [--seed 0]

Each case is a random model — ring soups (polyline or Catmull-Rom, random
ring sizes / segment counts / densities, near contacts that need refinement
or make curves intersect), closed random walks, or a mix — certified by
compute_linking_matrix and by the oracle (oracle/linkcert_oracle.py, pinned
to the reference).  Agreement: identical entries and pair lists, raw sums
within 1e-9, or the same DiscretizationError kind and loops.  Prints one JSON
summary line (and every mismatch).
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

import linkcert_oracle as oracle  # noqa: E402
import paper_2106_12655_b200 as lc  # noqa: E402
from paper_2106_12655_b200.certify import run_device_pipeline  # noqa: E402


def ring_soup(rng):
    count = int(rng.integers(2, 400))
    size = float(rng.uniform(max(1.5, 0.7 * count ** (1 / 3)), 15.0))   # fully interpenetrating soups take the
    # oracle (and the reference) many minutes of refinement passes
    n = int(rng.choice([5, 8, 12, 24, 48, 64, 100]))
    spline = bool(rng.random() < 0.35)
    loops = []
    th = 2 * np.pi * np.arange(n) / n
    for c in rng.uniform(0.0, size, size=(count, 3)):
        r = float(rng.uniform(0.3, 1.5))
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        v = np.cross(u, rng.normal(size=3))
        v /= np.linalg.norm(v)
        pts = c + r * (np.outer(np.cos(th), u) + np.outer(np.sin(th), v))
        if rng.random() < 0.3:
            pts = pts + 0.05 * r * rng.normal(size=pts.shape)
        loops.append(lc.LoopGeometry.from_catmull_rom(pts) if spline else lc.LoopGeometry.from_polyline(pts))
    return lc.CurveModel(loops), f"soup count={count} size={size:.2f} n={n} spline={spline}"


def walks(rng):
    count = int(rng.integers(2, 40))
    loops = []
    for _ in range(count):
        n = int(rng.integers(3, 200))
        pts = np.cumsum(rng.normal(size=(n, 3)), axis=0) * 0.5 + rng.uniform(0, 8, size=3)
        loops.append(lc.LoopGeometry.from_polyline(pts))
    return lc.CurveModel(loops), f"walks count={count}"


def with_contacts(rng):
    """A soup plus an exact copy of one ring (curves intersect) or a ring through
    another's vertex; or the soup under a tight pass / subsegment budget."""
    m, desc = ring_soup(rng)
    loops = list(m.loops)
    kind = int(rng.integers(0, 3))
    params = lc.DiscretizationParams()
    if kind == 0:
        k = int(rng.integers(0, len(loops)))
        loops.insert(int(rng.integers(0, len(loops) + 1)), loops[k])
        # every subsegment of the twins overlaps its copy, so the count doubles each
        # pass: a budget of a few thousand ends it in ~6 passes (the default 4M takes
        # the oracle -- and the reference -- many minutes of Python per pass)
        params = lc.DiscretizationParams(max_subsegments=int(rng.integers(1024, 16384)))
        desc += f" +duplicate ring subseg={params.max_subsegments}"
    elif kind == 1:
        k = int(rng.integers(0, len(loops)))
        v = loops[k].start_points()
        th = 2 * np.pi * np.arange(16) / 16
        pts = v[0] + 0.7 * (np.outer(np.cos(th), [0, 1, 0]) + np.outer(np.sin(th), [0, 0, 1])) - [0, 0.7, 0]
        pts[0] = v[0]   # exact contact: v0 + 0.7 - 0.7 can round 4e-16 off v0, which leaves a near-touching pair
        # whose Gauss sum is ill-conditioned (any summation order moves it by ~1e-3) instead of CurvesIntersect
        loops.append(lc.LoopGeometry.from_polyline(pts))   # passes through vertex 0 of ring k
        desc += " +ring through a vertex"
    else:
        params = lc.DiscretizationParams(max_passes=int(rng.integers(1, 4)),
                                         max_subsegments=int(rng.integers(4, 400)))
        desc += f" budget passes={params.max_passes} subseg={params.max_subsegments}"
    return (lc.CurveModel(loops), params), desc


def next_case(rng):
    u = rng.random()
    if u < 0.55:
        m, desc = ring_soup(rng)
        return m, desc, None
    if u < 0.7:
        m, desc = walks(rng)
        return m, desc, None
    (m, params), desc = with_contacts(rng)
    return m, desc, params


def run_case(m, params=None):
    params = params or lc.DiscretizationParams()
    coeffs, t, off = m.packed()
    try:
        pairs = oracle.pls(coeffs, t, off)
        verts, voff = oracle.discretize(coeffs, t, off, m.xi, pairs, params.epsilon, params.max_passes,
                                        params.max_subsegments)
        raw = oracle.evaluate_pairs(verts, voff, pairs)
        lk = np.array([oracle.round_link(r)[0] for r in raw], dtype=np.int64)
        keep = lk != 0
        want = np.concatenate([pairs[keep], lk[keep, None]], axis=1).astype(np.int64)
        o = ("ok", want, pairs, raw)
    except oracle.OracleDiscretizationError as e:
        o = ("err", e.kind, tuple(e.loops))
    t_oracle = time.time()
    try:
        got = lc.compute_linking_matrix(m, params=params)
        p2, r2, _, _, _ = run_device_pipeline(m, (), params)
        g = ("ok", got.array, np.array(p2).copy(), np.array(r2).copy())
    except lc.DiscretizationError as e:
        g = ("err", e.kind, tuple(e.loops))
    if o[0] != g[0]:
        return False, f"oracle {o[0]} vs gpu {g[0]}: {o[1:] if o[0] == 'err' else ''}{g[1:] if g[0] == 'err' else ''}"
    if o[0] == "err":
        return (o[1], o[2]) == (g[1], g[2]), f"errors {o[1:]} vs {g[1:]}"
    same = np.array_equal(o[1], g[1]) and np.array_equal(o[2], g[2])
    err = float(np.max(np.abs(o[3] - g[3]))) if len(o[3]) else 0.0
    ee_ok, ee_why = early_exit_case(m, params, o[1], o[2])
    return same and err < 1e-9 and ee_ok, f"entries equal={same} max raw err={err:.3g} {ee_why}"


def early_exit_case(m, params, want, pairs):
    """verify(early_exit=True) on a perturbed certificate (the oracle's entries with one
    flipped, one dropped, one added pair) against the reference's evaluation order
    replayed on the oracle's values (certify.py:195-216)."""
    import warnings

    rng = np.random.default_rng(len(want) * 7919 + len(pairs))
    ref = {(int(i), int(j)): int(v) for i, j, v in want}
    edits = []
    if ref:
        k = list(ref)[int(rng.integers(len(ref)))]
        ref[k] = -ref[k] if rng.random() < 0.5 else ref[k] + 1
        edits.append("changed")
    if len(ref) > 1 and rng.random() < 0.5:
        ref.pop(list(ref)[int(rng.integers(len(ref)))])
        edits.append("dropped")
    if m.num_loops > 3 and rng.random() < 0.5:
        i, j = sorted(rng.choice(m.num_loops, 2, replace=False).tolist())
        ref.setdefault((i, j), 3)
        edits.append("added")
    ref = {k: v for k, v in ref.items() if v != 0}   # a certificate stores no zero entries
    cert = lc.LinkMatrix(m.num_loops, tuple(sorted((i, j, v) for (i, j), v in ref.items())))
    values = {(int(i), int(j)): int(v) for i, j, v in want}
    cand = [(int(i), int(j)) for i, j in pairs]
    ordering = sorted(ref) + sorted(set(cand) - set(ref))
    first = next((p for p in ordering if values.get(p, 0) != ref.get(p, 0)), None)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        rep = lc.verify(m, cert, early_exit=True, params=params)
    ok = rep.first_failure == first and rep.status == ("Pass" if first is None else "Aborted")
    return ok, f"early exit {'+'.join(edits) or 'none'} first={first} got={rep.first_failure}"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--verbose", action="store_true", help="one line per case (model, outcome, seconds)")
    ap.add_argument("--budget", type=float, default=0.0, help="stop starting new cases after this many seconds")
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    t0 = time.time()
    stats = {"cases": 0, "agree": 0, "errors_agreed": 0, "mismatch": []}
    for k in range(args.cases):
        if args.budget and time.time() - t0 > args.budget:
            break
        m, desc, params = next_case(rng)
        t1 = time.time()
        try:
            ok, why = run_case(m, params)
        except Exception as exc:  # noqa: BLE001
            ok, why = False, f"exception {type(exc).__name__}: {exc}"
        if args.verbose:
            print(json.dumps({"case": k, "model": desc, "ok": ok, "why": why, "s": round(time.time() - t1, 2)}),
                  flush=True)
        stats["cases"] += 1
        if ok:
            stats["agree"] += 1
            stats["errors_agreed"] += why.startswith("errors")
        else:
            stats["mismatch"].append({"case": k, "model": desc, "why": why})
            print(json.dumps(stats["mismatch"][-1]), flush=True)
    stats["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(stats), flush=True)


if __name__ == "__main__":
    main()
