import sys, time, hashlib, os
sys.path.insert(0, '.')
import numpy as np
from paper_2106_12655_b200 import _native, generators as gen
m = gen.kusari_tube(after=True)
c, t, o = m.packed()
for nt in (1, 4, 8, 16):
    t0 = time.perf_counter(); b = _native.model_json(c, t, o, None, nt); t1 = time.perf_counter()
    print("format threads", nt, round(1e3 * (t1 - t0), 1), "ms", len(b))
data = bytes(b)
t0 = time.perf_counter(); h1, has = _native.sha256_hex(data); t1 = time.perf_counter()
print("native sha", round(1e3 * (t1 - t0), 1), "ms shani", has)
t0 = time.perf_counter(); hashlib.sha256(data).hexdigest(); print("hashlib", round(1e3 * (time.perf_counter() - t0), 1))
for nt in (4, 8, 16, 32):
    t0 = time.perf_counter(); _native.model_digest(c, t, o, None, nt); print("digest threads", nt, round(1e3 * (time.perf_counter() - t0), 1))
