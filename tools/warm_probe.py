"""verify() time on the Kusari tube, warm (cached snapshot) vs fresh model (GPU box):
    LC_DIGEST_STATS=1 python tools/warm_probe.py"""
import os, sys, time, warnings, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import generators as gen, workloads
before = gen.kusari_tube()
v, off = workloads.kusari_tube_vertices(after=True)
after = lc.CurveModel.from_polyline_arrays(v, off)
loops = [lc.LoopGeometry.from_polyline(v[off[k]:off[k + 1]]) for k in range(len(off) - 1)]
cert = lc.compute_linking_matrix(before)
warnings.simplefilter("ignore")
for name, mk in (("warm", lambda: after), ("fresh", lambda: lc.CurveModel(list(loops), xi=after.xi))):
    ts = []
    for r in range(12):
        m = mk()
        t0 = time.perf_counter(); lc.verify(m, cert); t1 = time.perf_counter()
        ts.append((t1 - t0) * 1e3)
    print(name, os.environ.get("LINKCERT_DIGEST_THREADS", "0"), "median", round(statistics.median(ts[2:]), 2),
          "min", round(min(ts[2:]), 2), flush=True)
