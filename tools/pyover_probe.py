import sys, time, statistics, os
os.environ.setdefault("LINKCERT_STAGE_TIMES", "1")   # every stage timed (diagnostic)
sys.path.insert(0, os.getcwd())
import torch
from paper_2106_12655_b200 import _native, generators as gen
from paper_2106_12655_b200.certify import device_step, excluded_keys, _dist
from paper_2106_12655_b200.direct import gauss_mode
from paper_2106_12655_b200.discretize import DiscretizationParams
from paper_2106_12655_b200.pls import upload
m = gen.kusari_tube(after=True); ctx = _native.context(0); upload(m, ctx)
ex, prm = excluded_keys(()), DiscretizationParams()
args = (ex, m.xi, prm.epsilon, prm.max_passes, prm.max_subsegments, gauss_mode())
for _ in range(5): device_step(ctx, m.xi, ex, prm)
def t(f, n=2000):
    t0 = time.perf_counter()
    for _ in range(n): f()
    return 1e6 * (time.perf_counter() - t0) / n
print("result_views us", t(ctx.result_views))
print("gauss_mode us", t(gauss_mode))
print("_dist us", t(_dist))
print("stage_times us", t(ctx.stage_times))
import numpy as np
print("ascontig us", t(lambda: np.ascontiguousarray(ex, dtype=np.uint64)))
ts=[]; tr=[]
for k in range(40):
    torch.cuda.synchronize(); t0=time.perf_counter(); ctx.run_pipeline(*args); t1=time.perf_counter(); ctx.result_views(); t2=time.perf_counter()
    ts.append(1e6*(t1-t0)); tr.append(1e6*(t2-t1))
print("run_pipeline us", statistics.median(ts[5:]), "views after run us", statistics.median(tr[5:]))
ts=[]
for k in range(40):
    torch.cuda.synchronize(); t0=time.perf_counter(); device_step(ctx, m.xi, ex, prm); ts.append(1e6*(time.perf_counter()-t0))
print("device_step us", statistics.median(ts[5:]), "b2r", ctx.stage_times()["begin_to_reduce"])
