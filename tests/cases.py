"""Named input models shared by tests/golden/make_golden.py and the tests.

Every model is built by paper_2106_12655_b200.generators; the fixtures store
a fingerprint of the packed arrays, so a test can assert it is evaluating
exactly the input the reference saw.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

from paper_2106_12655_b200 import generators as gen
from paper_2106_12655_b200.geometry import CurveModel, LoopGeometry


def fingerprint(model):
    coeffs, t, off = model.packed()
    h = hashlib.sha256()
    for a in (coeffs, t, off):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def circ(n, center, u, v, radius=1.0):
    t = np.linspace(0.0, 2.0 * math.pi, n, endpoint=False)
    return np.asarray(center, dtype=float) + radius * np.outer(np.cos(t), u) + radius * np.outer(np.sin(t), v)


def link_cases():
    cases = {"hopf1024": gen.hopf(1024)[0]}
    for T, P in [(1, 1), (1, 2), (1, 3), (1, 5), (2, 3), (3, 5), (10, 10)]:
        cases[f"torus_{T}_{P}_1024"] = gen.torus_link(T, P, 1024)[0]
    cases["torus_2_3_300"] = gen.torus_link(2, 3, 300)[0]
    cases["ribbon_10_2000"] = gen.double_helix_ribbon(10, 2000)[0]
    for seed in range(3):
        cases[f"perturbed_{seed}"] = gen.perturbed_random_link(seed=seed, n=200)[0]
    return cases


def cert_models(full=False):
    models = {
        "grid6": gen.square_link_grid(6)[0],
        "grid20": gen.square_link_grid(20)[0],
        "unlinked200": gen.unlinked_circles(200, 8)[0],
        "woundball3": gen.woundball(3)[0],
        "e4in1_8x8": gen.european_4in1(8, 8),
        "e4in1_32x32": gen.european_4in1(32, 32),
        "kusari_small": gen.kusari_tube(n_around=12, rows=4, partial=5),
        "knit_6_8_800": gen.knit_tube(courses=6, n=800, W=8),
        "spline_perturbed_5": gen.perturbed_random_link(T=2, P=3, n=96, seed=5, spline=True)[0],
        "spline_perturbed_3": gen.perturbed_random_link(T=1, P=2, n=48, seed=3, spline=True)[0],
    }
    if full:
        models["kusari_full"] = gen.kusari_tube()
    return models


def edit_cases(full=False):
    """name -> (before, after) models for verify (pull-through detection)."""
    g, _ = gen.square_link_grid(6)
    pts = [lp.start_points() for lp in g.loops]
    pts[2] = pts[2] + np.array([0.0, 0.0, 50.0])
    ks = gen.kusari_tube(n_around=12, rows=4, partial=5)
    n_big = 12 * 4 + 5
    kpts = [lp.control_points.copy() for lp in ks.loops]
    kpts[n_big + 3] = kpts[n_big + 3] + np.array([0.0, 0.0, 100.0])
    kpts[n_big + 5] = kpts[n_big + 5][::-1].copy()
    edits = {
        "grid6_pull": (g, CurveModel([LoopGeometry.from_polyline(p) for p in pts])),
        "e4in1_32x32_pull165": (gen.european_4in1(32, 32), gen.european_4in1(32, 32, moved={165: 3.0})),
        "kusari_small_after": (ks, CurveModel([LoopGeometry.from_polyline(p) for p in kpts])),
    }
    if full:
        edits["kusari_full_after"] = (gen.kusari_tube(), gen.kusari_tube(after=True))
    return edits


def disc_error_cases():
    """name -> (model, pairs, DiscretizationParams kwargs) (test_discretize.py:90-123)."""
    ex, ey, ez = np.eye(3)

    def spline(p):
        return LoopGeometry.from_catmull_rom(p)

    a = spline(circ(16, (0, 0, 0), ex, ey))
    b = spline(circ(16, (1.0, 0, 0), ez, ex))
    c = spline(circ(16, (1.0, 0, 0), ez, ey))
    tight = CurveModel([spline(circ(12, (0, 0, 0), ex, ey)), spline(circ(12, (1.9, 0, 0), ez, ex))])
    p8 = circ(8, (0, 0, 0), ex, ey)
    zero = CurveModel([LoopGeometry.from_polyline(circ(8, (1.0, 0, 0), ex, ey)),
                       LoopGeometry.from_polyline(np.vstack([p8, p8[-1:]]))])
    return {
        "intersect": (CurveModel([a, b, c]), [(0, 1), (0, 2), (1, 2)], {}),
        "tight_ok": (tight, [(0, 1)], {}),
        "tight_one_pass": (tight, [(0, 1)], {"max_passes": 1}),
        "tight_budget": (tight, [(0, 1)], {"max_subsegments": 1}),
        "zero_length": (zero, [(0, 1)], {}),
    }


def _returning_loop(off):
    """Closed 4-segment cubic loop whose first segment returns to its start
    point (non-degenerate tight box, zero-length chord)."""
    p0, p1, p2 = (np.array(v, dtype=np.float64) + off for v in ([0, 0, 0], [4, 0, 0], [2, 3, 0]))
    c = np.zeros((4, 4, 3))
    c[0, 0], c[0, 1], c[0, 2], c[0, 3] = p0, [3, 0, 1], [-3, 3, 0], [0, -3, -1]
    c[1, 0], c[1, 1] = p0, p1 - p0
    c[2, 0], c[2, 1] = p1, p2 - p1
    c[3, 0], c[3, 1] = p2, p0 - p2
    return LoopGeometry(c)


def validation_cases():
    """name -> model whose chords fail PolylineLoop validation with no refinement
    pass (compute_linking_matrix raises ValidationError): unpaired and paired."""
    def tri(off, s=1.0):
        return LoopGeometry.from_polyline(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0.0]]) * s + np.asarray(off))

    return {
        "returning_unpaired": CurveModel([_returning_loop(np.zeros(3)), tri([50.0, 0.0, 0.0])]),
        "returning_paired": CurveModel([_returning_loop(np.zeros(3)), tri([1.5, 1.0, 0.1], 0.3)]),
    }
