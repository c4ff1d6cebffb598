import sys, time, statistics, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native, generators as gen
a, b = gen.torus_pair(2, 3, 1024)
ctx = _native.context()
def med(f, n=40):
    ts = []
    for k in range(n + 5):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts[5:]) * 1e6, 1)
print("lc.link_direct us", med(lambda: lc.link_direct(a, b)))
print("ctx.link_direct us", med(lambda: ctx.link_direct(a, b)))
lc.link_direct(a, b); print("gauss kernel ms", ctx.last_gauss_ms())
import numpy as np
a3 = np.ascontiguousarray(a); b3 = np.ascontiguousarray(b)
print("ctx.link_direct (contig) us", med(lambda: ctx.link_direct(a3, b3)))
