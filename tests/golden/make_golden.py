"""Generate golden vectors by running the REFERENCE linkcert package (this container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py [--full]

Inputs come from tests/cases.py (paper_2106_12655_b200.generators; packed
arrays fingerprinted in the fixtures); every expected value comes from
/root/reference/pkg/src/linkcert.  Nothing is written outside tests/golden/.
--full adds the Kusari-scale C3 tube (~1 min of reference time).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import warnings
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, "/root/reference/pkg/src")

import linkcert as ref  # noqa: E402
from linkcert.discretize import DiscretizationError as RefDiscErr  # noqa: E402

import cases  # noqa: E402
from cases import fingerprint  # noqa: E402


def ref_fingerprint(model):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(np.concatenate([lp.coeffs for lp in model.loops])).tobytes())
    h.update(np.ascontiguousarray(np.concatenate([lp.t for lp in model.loops])).tobytes())
    off = np.zeros(model.num_loops + 1, dtype=np.int64)
    np.cumsum([len(lp) for lp in model.loops], out=off[1:])
    h.update(off.tobytes())
    return h.hexdigest()


def to_ref(model):
    """Our CurveModel -> reference CurveModel with identical arrays (and identical xi)."""
    loops = []
    for lp in model.loops:
        if lp.is_polyline and np.all(lp.t[:, 0] == 0) and np.all(lp.t[:, 1] == 1):
            loops.append(ref.LoopGeometry.from_polyline(lp.control_points))
        else:
            loops.append(ref.LoopGeometry(lp.coeffs, lp.t, closed=lp.closed, control_points=lp.control_points))
    rm = ref.CurveModel(loops)
    assert rm.xi == model.xi, (rm.xi, model.xi)
    assert ref_fingerprint(rm) == fingerprint(model)
    return rm


def entries_of(matrix):
    return np.array(matrix.entries, dtype=np.int64).reshape(-1, 3)


def report_dict(r):
    return {"status": r.status, "destroyed": [list(p) for p in r.destroyed], "created": [list(p) for p in r.created],
            "changed": [list(p) for p in r.changed],
            "first_failure": list(r.first_failure) if r.first_failure else None}


def main(full=False):
    out_json = {}
    arrays = {}

    # 1. segment-pair lambdas (direct.py:137-146), incl. near-degenerate geometry
    rng = np.random.default_rng(12655)
    q = rng.normal(size=(2000, 12))
    q[1000:1200, 9:12] = q[1000:1200, 6:9] + 1e-9 * rng.normal(size=(200, 3))     # tiny outer segment
    q[1200:1400, 2] = q[1200:1400, 5] = q[1200:1400, 8] = q[1200:1400, 11] = 0.0  # coplanar (p == 0)
    q[1400:1600, 3:6] = q[1400:1600, 0:3] * 1.0000001                              # tiny inner segment
    q[1600:1800] *= 1e6
    q[1800:2000] *= 1e-6
    arrays["quads"] = q
    arrays["quads_lambda"] = np.array([ref.segment_pair_lambda(r[0:3], r[3:6], r[6:9], r[9:12]) for r in q])

    # 2. link_direct raw values (atan + anglesum) on C1 and the test_direct cases
    links = {}
    for name, m in cases.link_cases().items():
        rm = to_ref(m)
        a, b = (lp.start_points() for lp in rm.loops)
        links[name] = {"fingerprint": fingerprint(m), "atan": ref.link_direct(a, b, "atan"),
                       "anglesum": ref.link_direct(a, b, "anglesum"), "atan_swapped": ref.link_direct(b, a, "atan")}
    # random (self-intersecting) polygons: exercises every sign / wrap branch
    for k in range(4):
        a = rng.normal(size=(17 + 13 * k, 3))
        b = rng.normal(size=(23 + 7 * k, 3)) + 0.25
        arrays[f"rand_a{k}"] = a
        arrays[f"rand_b{k}"] = b
        links[f"random_{k}"] = {"atan": ref.link_direct(a, b, "atan"), "anglesum": ref.link_direct(a, b, "anglesum")}
    out_json["links"] = links

    # 3. certificates, PLS pairs and discretized vertices on every config family
    certs = {}
    for name, m in cases.cert_models(full).items():
        rm = to_ref(m)
        pairs = np.array(ref.potential_link_search(rm).pairs, dtype=np.int64).reshape(-1, 2)
        mat = ref.compute_linking_matrix(rm)
        arrays[f"{name}__pairs"] = pairs
        arrays[f"{name}__entries"] = entries_of(mat)
        polys = ref.discretize(rm, ref.potential_link_search(rm))
        nverts = [len(p) for p in polys]
        vh = hashlib.sha256(np.concatenate([p.vertices for p in polys]).tobytes()).hexdigest()
        certs[name] = {"fingerprint": fingerprint(m), "xi": rm.xi, "digest": ref.model_digest(rm),
                       "num_pairs": len(pairs), "num_links": len(mat.entries),
                       "discretized_vertices": int(sum(nverts)), "discretized_sha256": vh}
        if sum(nverts) <= 20000:
            arrays[f"{name}__verts"] = np.concatenate([p.vertices for p in polys])
            arrays[f"{name}__vert_off"] = np.concatenate([[0], np.cumsum(nverts)]).astype(np.int64)
        print(name, certs[name], flush=True)
    out_json["certs"] = certs

    # 4. verify before/after edits (pull-through detection), incl. early exit
    reports = {}
    for name, (before, after) in cases.edit_cases(full).items():
        rb, ra = to_ref(before), to_ref(after)
        cert = ref.compute_linking_matrix(rb)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            rep = ref.verify(ra, cert)
            rep_ee = ref.verify(ra, cert, early_exit=True)
        arrays[f"{name}__after_entries"] = entries_of(ref.compute_linking_matrix(ra))
        reports[name] = {"before_fingerprint": fingerprint(before), "after_fingerprint": fingerprint(after),
                         "full": report_dict(rep), "early_exit": report_dict(rep_ee),
                         "after_digest": ref.model_digest(ra)}
        print(name, reports[name]["full"], reports[name]["early_exit"]["first_failure"], flush=True)
    out_json["verify"] = reports

    # 5. discretization error cases (test_discretize.py:90-123)
    errs = {}
    for name, (m, prs, kw) in cases.disc_error_cases().items():
        rm = to_ref(m)
        try:
            polys = ref.discretize(rm, ref.PairList(tuple(prs)), ref.DiscretizationParams(**kw))
            errs[name] = {"ok": True, "nverts": [len(p) for p in polys]}
            arrays[f"disc_{name}__verts"] = np.concatenate([p.vertices for p in polys])
        except RefDiscErr as e:
            errs[name] = {"ok": False, "kind": e.kind, "loops": list(e.loops), "message": str(e)}
        errs[name]["fingerprint"] = fingerprint(m)
        errs[name]["pairs"] = prs
        errs[name]["params"] = kw
        print(name, errs[name], flush=True)
    out_json["discretize"] = errs

    # 6. chord validation errors through the whole pipeline
    vals = {}
    for name, m in cases.validation_cases().items():
        rm = to_ref(m)
        try:
            ref.compute_linking_matrix(rm)
            vals[name] = {"ok": True}
        except ref.ValidationError as e:
            vals[name] = {"ok": False, "message": str(e)}
        vals[name]["fingerprint"] = fingerprint(m)
        vals[name]["pairs"] = [list(p) for p in ref.potential_link_search(rm)]
        print(name, vals[name], flush=True)
    out_json["validation"] = vals

    with open(HERE / "golden.json", "w") as f:
        json.dump(out_json, f, indent=1, sort_keys=True)
    np.savez_compressed(HERE / "golden_arrays.npz", **arrays)
    print("wrote", HERE / "golden.json", HERE / "golden_arrays.npz")


if __name__ == "__main__":
    main(full="--full" in sys.argv)
