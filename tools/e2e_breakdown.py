"""Where does verify() spend its time on the Kusari tube?  (GPU box)
A fresh CurveModel each repetition (loops built one by one, outside the timers)."""
import os, sys, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import generators as gen, _native, model_io, pls, workloads
from paper_2106_12655_b200.certify import device_step, diff_arrays, excluded_keys
before = gen.kusari_tube()
v, off = workloads.kusari_tube_vertices(after=True)
loops = [lc.LoopGeometry.from_polyline(v[off[k]:off[k + 1]]) for k in range(len(off) - 1)]
xi = lc.CurveModel.from_polyline_arrays(v, off).xi
cert = lc.compute_linking_matrix(before)
ctx = _native.context()
for rep in range(5):
    t = {}
    m = lc.CurveModel(list(loops), xi=xi)
    t0 = time.perf_counter(); snap = m.snapshot(); t["snapshot"] = time.perf_counter() - t0
    t0 = time.perf_counter(); d = model_io.model_digest(m, snap); t["digest"] = time.perf_counter() - t0
    t0 = time.perf_counter(); pls.upload(m, ctx, snap); t["upload"] = time.perf_counter() - t0
    t0 = time.perf_counter(); res = device_step(ctx, m.xi, excluded_keys(()), lc.DiscretizationParams()); t["device_step"] = time.perf_counter() - t0
    t0 = time.perf_counter(); rep_ = diff_arrays(cert.array, *res); t["diff"] = time.perf_counter() - t0
    m = lc.CurveModel(list(loops), xi=xi)
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore"); r = lc.verify(m, cert)
    t["verify_total_fresh"] = time.perf_counter() - t0
    print({k: round(val * 1e3, 2) for k, val in t.items()}, os.cpu_count(), flush=True)
