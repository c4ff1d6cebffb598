"""Full BASELINE config C4 on one GPU: 200 knit courses x 100k segments (1.99e12 seg-pairs).
Checks the certificate (199 adjacent pairs, LK = -100 each) and times it (GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import generators as gen
t0 = time.perf_counter()
m = gen.knit_tube(courses=200, n=100_000, W=100)
t1 = time.perf_counter()
timings = {}
mat = lc.compute_linking_matrix(m, timings=timings)
t2 = time.perf_counter()
arr = mat.array
ok = len(arr) == 199 and np.all(arr[:, 1] == arr[:, 0] + 1) and np.all(arr[:, 2] == -100)
print(f"build {t1 - t0:.1f} s, certificate {t2 - t1:.2f} s, entries {len(arr)}, all adjacent LK=-100: {ok}")
print({k: round(v, 4) for k, v in timings.items()})
sp = 199 * 100_000 ** 2
print(f"seg-pairs {sp:.3e} -> {sp / timings['kernel']:.3e} seg-pairs/s (kernel stage)")
