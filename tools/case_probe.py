"""Time the CUDA path on one fuzz case (tools/fuzz_parity.py generator order).

    python tools/case_probe.py --seed 2 --case 14
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

import fuzz_parity as f  # noqa: E402
import paper_2106_12655_b200 as lc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seed", type=int, default=2)
ap.add_argument("--case", type=int, default=14)
args = ap.parse_args()
rng = np.random.default_rng(args.seed)
for k in range(args.case + 1):
    m, desc, params = f.next_case(rng)
print(desc, m.num_loops, flush=True)
t0 = time.time()
try:
    mat = lc.compute_linking_matrix(m, params=params)
    print("ok", len(mat.entries), round(time.time() - t0, 2), "s", flush=True)
except lc.DiscretizationError as e:
    print("error", e.kind, e.loops[:10], round(time.time() - t0, 2), "s", flush=True)
