"""Small end-to-end run of every device path for compute-sanitizer (GPU box):
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_probe.py
Fused path (first run uncaptured, then captured and replayed as a CUDA graph),
staged path (LINKCERT_FUSED=0 inside), refinement (spline rings), anglesum,
device early exit, PLS sweep, Barnes-Hut; each result checked against the first."""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2106_12655_b200 as lc  # noqa: E402
from paper_2106_12655_b200 import _native, generators as gen  # noqa: E402

warnings.simplefilter("ignore")
before = gen.kusari_tube(n_around=12, rows=4, partial=5)
pts = [lp.control_points.copy() for lp in before.loops]
pts[60] = pts[60][::-1].copy()
after = lc.CurveModel([lc.LoopGeometry.from_polyline(p) for p in pts])
ctx = _native.context()
cert = lc.compute_linking_matrix(before)
paths = []
for k in range(3):   # uncaptured, captured, replayed
    rep = lc.verify(after, cert)
    paths.append(ctx.last_run_fused())
    assert rep.status == "Fail" and rep.changed
full = rep
ee = lc.verify(after, cert, early_exit=True)
assert ee.status == "Aborted" and ee.first_failure in full.changed
os.environ["LINKCERT_FUSED"] = "0"
assert lc.verify(after, cert) == full
os.environ.pop("LINKCERT_FUSED")
os.environ["LINKCERT_PLS_SWEEP"] = "1"
assert lc.verify(after, cert, early_exit=False) == full
os.environ.pop("LINKCERT_PLS_SWEEP")
an = lc.compute_linking_matrix(before, choice=lc.KernelChoice(ds_variant="anglesum"))
assert np.array_equal(an.array, cert.array)
rng = np.random.default_rng(3)
th = 2 * np.pi * np.arange(12) / 12
rings = []
for c in rng.uniform(0.0, 4.0, size=(30, 3)):
    u = rng.normal(size=3)
    u /= np.linalg.norm(u)
    v = np.cross(u, rng.normal(size=3))
    v /= np.linalg.norm(v)
    rings.append(lc.LoopGeometry.from_catmull_rom(c + np.outer(np.cos(th), u) + np.outer(np.sin(th), v)))
spl = lc.CurveModel(rings)
try:
    m = lc.compute_linking_matrix(spl)
    print("spline soup entries", len(m.entries))
except lc.DiscretizationError as exc:
    print("spline soup:", exc)
a, b = gen.ribbon_pair(5, 2000)
bh = lc.barnes_hut_detailed(lc.build_moment_tree(lc.PolylineLoop(a)), lc.build_moment_tree(lc.PolylineLoop(b)))
assert abs(bh.value - 5) < 0.05
print("sanitize probe ok; fused paths", paths)
