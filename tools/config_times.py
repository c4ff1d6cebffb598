"""Per-config timings on the GPU box (not bench lines): C1 link_direct on 1024 x 1024
torus links, C2 European 4-in-1 32 x 32 (device step and fresh-model verify), C3 the
Kusari tube (device step).  python tools/config_times.py"""
import os, statistics, sys, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native, generators as gen
from paper_2106_12655_b200.certify import device_step, excluded_keys
from paper_2106_12655_b200.discretize import DiscretizationParams
from paper_2106_12655_b200.pls import upload

warnings.simplefilter("ignore")
ctx = _native.context(0)


def med(f, n=30, warm=5):
    ts = []
    for k in range(n + warm):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        if k >= warm:
            ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts)


m, _ = gen.hopf(1024)
c1 = {"hopf": (m.loops[0].control_points, m.loops[1].control_points)}
for T, P in ((2, 3), (10, 10)):
    c1[f"torus({T},{P})"] = gen.torus_pair(T, P, 1024)
for name, (a, b) in c1.items():
    raw = lc.link_direct(a, b)
    print(f"C1 {name} 1024 x 1024: link_direct {med(lambda: lc.link_direct(a, b)):.3f} ms (host wall), raw {raw:.15f}")

for name, (before, after) in (("C2 e4in1 32x32", (gen.european_4in1(32, 32), gen.european_4in1(32, 32, moved={165: 3.0}))),
                              ("C3 Kusari tube", (gen.kusari_tube(), gen.kusari_tube(after=True)))):
    cert = lc.compute_linking_matrix(before)
    upload(after, ctx)
    ex, prm = excluded_keys(()), DiscretizationParams()
    step = med(lambda: device_step(ctx, after.xi, ex, prm))
    loops = [lc.LoopGeometry.from_polyline(lp.control_points) for lp in after.loops]
    ver = med(lambda: lc.verify(lc.CurveModel(list(loops), xi=after.xi), cert), n=10, warm=2)
    P = len(lc.potential_link_search(after))
    print(f"{name}: L={after.num_loops} P={P} entries={len(cert.entries)}: device step {step:.3f} ms (host wall, "
          f"sync'd), verify (fresh model, incl. digest) {ver:.2f} ms")
