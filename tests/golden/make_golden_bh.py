"""Generate Barnes-Hut golden vectors by running the REFERENCE linkcert package
(this container only; /root/reference does not exist on the GPU box).

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden_bh.py

Every input array is stored next to the expected values (bh_golden.npz), so the
tests never regenerate geometry.  Expected values come from
/root/reference/pkg/src/linkcert (barneshut.py, bvh.py, kernels.py, certify.py).
"""

from __future__ import annotations

import json
import math
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
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import linkcert as ref  # noqa: E402
from linkcert import generators as rgen  # noqa: E402
from linkcert.barneshut import MomentNode  # noqa: E402

import cases  # noqa: E402
from make_golden import entries_of, to_ref  # noqa: E402

TREE_FIELDS = ("node_lo", "node_hi", "left", "right", "start", "end", "prim_order")
MOMENT_FIELDS = ("center", "radius", "cm", "cd", "cq", "ncm", "ncd", "ncq")


def circle_points(n, center=(0.0, 0.0, 0.0), u=(1.0, 0.0, 0.0), v=(0.0, 1.0, 0.0), radius=1.0):
    t = np.linspace(0.0, 2.0 * math.pi, n, endpoint=False)
    return (np.asarray(center, dtype=float) + radius * np.outer(np.cos(t), np.asarray(u, dtype=float))
            + radius * np.outer(np.sin(t), np.asarray(v, dtype=float)))


def tree_loops():
    rng = np.random.default_rng(2)
    loops = {
        "circle16": circle_points(16, radius=2.0),
        "noisy64": circle_points(64, radius=3.0) + 0.2 * rng.normal(size=(64, 3)),
        "circle33": circle_points(33, radius=7.0, center=(4.0, 1.0, -2.0)),
        "circle50": circle_points(50),
    }
    # integer zig-zag: many equal segment centers on every axis (tie breaking by index)
    zz = []
    for k in range(24):
        zz.append((k % 4, (k // 4) % 3, (k * 7) % 5))
    loops["ties24"] = np.asarray(zz, dtype=float)
    loops["single3"] = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    model, _ = rgen.double_helix_ribbon(5, 300)
    loops["helix300"] = model.loops[0].start_points()
    rng7 = np.random.default_rng(7)
    loops["random400"] = np.cumsum(rng7.normal(size=(400, 3)), axis=0)
    return loops


def arc_pair(dist):
    rng = np.random.default_rng(6)
    t = np.linspace(0.0, 1.0, 40)
    arc1 = np.stack([t, 0.3 * np.sin(7 * t), 0.2 * np.cos(5 * t)], axis=1)
    arc1 += 0.01 * rng.normal(size=arc1.shape)
    arc2 = arc1[::-1] * np.array([1.0, -1.0, 1.0])
    p1 = np.vstack([arc1, arc1[::-1] + [0.0, 0.0, 1.5]])
    p2 = np.vstack([arc2, arc2[::-1] + [0.0, 1.5, 0.0]]) + np.array([dist, dist, dist]) / np.sqrt(3)
    return p1, p2


def bh_cases():
    c = {}
    c["hopf32"] = (circle_points(32), circle_points(32, center=(1.0, 0.0, 0.0), u=(0.0, 0.0, 1.0), v=(1.0, 0.0, 0.0)),
                   {})
    m, _ = rgen.torus_link(2, 3, n=256)
    c["torus23_beta1e6"] = (m.loops[0].start_points(), m.loops[1].start_points(),
                            dict(beta_init=1e6, beta_max=1e6, adaptive=False))
    m, _ = rgen.double_helix_ribbon(5, 1200)
    a, b = (lp.start_points() for lp in m.loops)
    for beta in (2.0, 8.0, 32.0):
        c[f"ribbon5_beta{int(beta)}"] = (a, b, dict(beta_init=beta, beta_max=beta, adaptive=False))
    m, _ = rgen.double_helix_ribbon(8, 1500)
    a, b = (lp.start_points() for lp in m.loops)
    c["ribbon8_fixed1"] = (a, b, dict(beta_init=1.0, beta_max=1.0, adaptive=False))
    c["ribbon8_adaptive"] = (a, b, dict(beta_init=1.0, beta_max=10.0, e_target=1e-3))
    m, _ = rgen.torus_link(3, 5, n=400)
    a, b = (lp.start_points() for lp in m.loops)
    c["torus35_default"] = (a, b, {})
    c["torus35_dipole"] = (a, b, dict(order="dipole"))
    p1, p2 = arc_pair(5.0)
    c["arcs_far"] = (p1, p2, {})
    rng = np.random.default_rng(11)
    w1 = circle_points(200, radius=2.0) + 0.05 * rng.normal(size=(200, 3))
    w2 = circle_points(180, center=(2.0, 0.0, 0.0), u=(0.0, 0.0, 1.0), v=(1.0, 0.0, 0.0), radius=2.0)
    c["wobbly_hopf"] = (w1, w2, dict(e_target=0.01))
    c["self_pair"] = (w1, w1, dict(adaptive=False))
    return c


def main():
    arrays, meta = {}, {"trees": [], "far_field": [], "bh": [], "matrices": {}}
    for name, pts in tree_loops().items():
        tree = ref.build_moment_tree(pts)
        arrays[f"tree_{name}_verts"] = np.asarray(pts, dtype=np.float64)
        for f in TREE_FIELDS:
            arrays[f"tree_{name}_{f}"] = getattr(tree.bvh, f)
        for f in MOMENT_FIELDS:
            arrays[f"tree_{name}_{f}"] = getattr(tree, f)
        arrays[f"tree_{name}_loop_length"] = np.array([tree.loop_length])
        meta["trees"].append(name)

    # far-field values: arcs at three distances, depth-2 nodes (test_barneshut.py:58-84)
    ff = []
    for dist in (20.0, 40.0, 80.0):
        p1, p2 = arc_pair(dist)
        t1, t2 = ref.build_moment_tree(p1), ref.build_moment_tree(p2)
        for na in range(min(7, t1.bvh.num_nodes)):
            for nb in range(min(7, t2.bvh.num_nodes)):
                for order in ("dipole", "quadrupole"):
                    v = ref.far_field_eval(MomentNode(t1, na), MomentNode(t2, nb), order)
                    ff.append((dist, na, nb, 1 if order == "quadrupole" else 0, v))
        arrays[f"ff_{int(dist)}_a"] = p1
        arrays[f"ff_{int(dist)}_b"] = p2
    arrays["ff_values"] = np.array(ff, dtype=np.float64)

    for name, (a, b, kw) in bh_cases().items():
        params = ref.BarnesHutParams(**kw)
        r = ref.barnes_hut_detailed(ref.build_moment_tree(a), ref.build_moment_tree(b), params)
        arrays[f"bh_{name}_a"] = np.asarray(a, dtype=np.float64)
        arrays[f"bh_{name}_b"] = np.asarray(b, dtype=np.float64)
        meta["bh"].append({"name": name, "params": kw, "value": r.value, "e_estimate": r.e_estimate,
                           "beta_used": r.beta_used, "reran": r.reran,
                           "direct": ref.link_direct(np.asarray(a), np.asarray(b))})
        print(name, r, flush=True)

    # certificates with the Barnes-Hut kernel (certify.py:141-166 via kernels.py:45-73)
    choice = ref.KernelChoice(method="bh")
    from paper_2106_12655_b200 import generators as ours
    models = {"grid4": ours.square_link_grid(4)[0], "e4in1_6x6": ours.european_4in1(6, 6),
              "kusari_small": ours.kusari_tube(n_around=12, rows=4, partial=5)}
    tight = {"e4in1_6x6"}   # also with a tight error target: per-pair reruns with their own beta
    runs = [(n, m, choice, {}) for n, m in models.items()]
    runs += [(n + "_tight", models[n], ref.KernelChoice(method="bh", bh=ref.BarnesHutParams(e_target=1e-4)),
              {"e_target": 1e-4}) for n in tight]
    for name, model, choice, kw in runs:
        rm = to_ref(model)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            mat = ref.compute_linking_matrix(rm, choice=choice)
        arrays[f"mat_{name}_entries"] = entries_of(mat)
        meta["matrices"][name] = {"kernel_tag": mat.kernel_tag, "digest": mat.model_digest, "bh_params": kw,
                                  "model": name.replace("_tight", ""),
                                  "fingerprint": cases.fingerprint(model),
                                  "diagnostics": {f"{i},{j}": d for (i, j), d in mat.diagnostics.items()}}
        print(name, len(mat.entries), len(mat.diagnostics), flush=True)

    np.savez_compressed(HERE / "bh_golden.npz", **arrays)
    (HERE / "bh_golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
