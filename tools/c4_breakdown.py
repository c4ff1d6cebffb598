"""C4 (200 knit courses x 100k) certificate: where the time goes (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import generators as gen, model_io, pls, _native
from paper_2106_12655_b200.certify import device_step, excluded_keys
t0 = time.perf_counter(); m = gen.knit_tube(courses=200, n=100_000, W=100); t1 = time.perf_counter()
print(f"build {t1 - t0:.2f} s", flush=True)
ctx = _native.context()
for rep in range(2):
    t = {}
    m2 = lc.CurveModel(list(m.loops), xi=m.xi)
    a = time.perf_counter(); snap = m2.snapshot(); t["snapshot"] = time.perf_counter() - a
    a = time.perf_counter(); d = model_io.model_digest(m2, snap); t["digest"] = time.perf_counter() - a
    a = time.perf_counter(); pls.upload(m2, ctx, snap); ctx.synchronize(); t["upload"] = time.perf_counter() - a
    tm = {}
    a = time.perf_counter(); res = device_step(ctx, m2.xi, excluded_keys(()), lc.DiscretizationParams(), timings=tm)
    t["device_step"] = time.perf_counter() - a
    m3 = lc.CurveModel(list(m.loops), xi=m.xi)
    a = time.perf_counter(); mat = lc.compute_linking_matrix(m3); t["certificate_total"] = time.perf_counter() - a
    print({k: round(v, 3) for k, v in t.items()}, {k: round(v, 3) for k, v in tm.items()}, "path", ctx.last_run_fused(),
          flush=True)
