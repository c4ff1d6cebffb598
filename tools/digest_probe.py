"""Digest pipeline timing on the GPU box host (LC_DIGEST_STATS=1: hasher wait/hash split)."""
import os, sys, time
os.environ["LC_DIGEST_STATS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_12655_b200 import _native, generators as gen
m = gen.kusari_tube(after=True)
c, t, o = m.packed()
blob = bytes(_native.model_json(c, t, o, None, 16))
for rep in range(2):
    t0 = time.perf_counter(); _native.sha256_hex(blob); print("sha alone", round(1e3 * (time.perf_counter() - t0), 2), flush=True)
for nt in (2, 3, 4, 6, 8, 12, 16):
    for rep in range(2):
        t0 = time.perf_counter(); _native.model_digest(c, t, o, None, nt)
        print("digest nt", nt, round(1e3 * (time.perf_counter() - t0), 2), flush=True)
