"""Models that need refinement passes (the staged path): certificate time per call (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native, generators as gen


def spline_sheet(rows=32, cols=32, npts=15):
    c, us, vs = gen.european_4in1_params(rows, cols)
    th = 2 * np.pi * np.arange(npts) / npts
    return lc.CurveModel([lc.LoopGeometry.from_catmull_rom(c[k] + np.outer(np.cos(th), us[k]) + np.outer(np.sin(th), vs[k]))
                          for k in range(rows * cols)])


def soup(seed, count, size, spline):
    rng = np.random.default_rng(seed)
    th = 2 * np.pi * np.arange(24) / 24
    loops = []
    for c in rng.uniform(0.0, size, size=(count, 3)):
        u = rng.normal(size=3); u /= np.linalg.norm(u)
        v = np.cross(u, rng.normal(size=3)); v /= np.linalg.norm(v)
        pts = c + np.outer(np.cos(th), u) + np.outer(np.sin(th), v)
        loops.append(lc.LoopGeometry.from_catmull_rom(pts) if spline else lc.LoopGeometry.from_polyline(pts))
    return lc.CurveModel(loops)


for name, m in [("spline_sheet_32x32", spline_sheet()), ("soup_400_poly", soup(1, 400, 12.0, False)),
                ("soup_4000_spline", soup(2, 4000, 26.0, True))]:
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        timings = {}
        mat = lc.compute_linking_matrix(m, timings=timings)
        ts.append(time.perf_counter() - t0)
    polys = lc.discretize(m, lc.potential_link_search(m))
    nv = sum(len(p) for p in polys)
    print(f"{name}: loops {m.num_loops} links {len(mat.entries)} chord verts {nv} (segments "
          f"{sum(lp.coeffs.shape[0] for lp in m.loops)}) path {_native.context().last_run_fused()} "
          f"best {1e3 * min(ts):.2f} ms timings {dict((k, round(1e3 * v, 3)) for k, v in timings.items())}", flush=True)
