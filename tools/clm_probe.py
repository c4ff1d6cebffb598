import sys, time, statistics, os, warnings
sys.path.insert(0, os.getcwd())
warnings.simplefilter("ignore")
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native, generators as gen
m, _ = gen.hopf(1024)
ctx = _native.context()
def med(f, n=20):
    ts = []
    for k in range(n + 3):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts[3:]) * 1e3, 3)
print("compute_linking_matrix(hopf 1024) ms", med(lambda: lc.compute_linking_matrix(m)))
print("path", ctx.last_run_fused())
print(ctx.stage_times())
