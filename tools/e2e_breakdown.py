"""Where does verify() spend its time on the Kusari tube?  (GPU box)"""
import os, sys, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import generators as gen, _native, model_io, pls
from paper_2106_12655_b200.certify import device_step, diff_arrays, excluded_keys
before, after = gen.kusari_tube(), gen.kusari_tube(after=True)
cert = lc.compute_linking_matrix(before)
ctx = _native.context()
for rep in range(3):
    t = {}
    t0 = time.perf_counter(); d = model_io.model_digest(after); t["digest"] = time.perf_counter() - t0
    t0 = time.perf_counter(); pls.upload(after); t["upload"] = time.perf_counter() - t0
    t0 = time.perf_counter(); res = device_step(ctx, after.xi, excluded_keys(()), lc.DiscretizationParams()); t["device_step"] = time.perf_counter() - t0
    t0 = time.perf_counter(); rep_ = diff_arrays(cert.array, *res); t["diff"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore"); r = lc.verify(after, cert)
    t["verify_total"] = time.perf_counter() - t0
    print({k: round(v * 1e3, 2) for k, v in t.items()}, os.cpu_count(), flush=True)
