"""Profiling driver (run under ncu on the GPU box; never a bench number).

  python tools/prof_gauss.py --case kusari --mode phase --reps 2
  python tools/prof_gauss.py --case torus --mode ref --reps 1     # F_pair: dynamic FP64 ops / pair
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2106_12655_b200 import _native, generators as gen  # noqa: E402
from paper_2106_12655_b200.certify import device_step, excluded_keys  # noqa: E402
from paper_2106_12655_b200.discretize import DiscretizationParams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="kusari", choices=["kusari", "torus", "ribbon"])
    ap.add_argument("--mode", default="phase", choices=list(_native.GAUSS_MODES) + ["anglesum"])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--n", type=int, default=1024)
    a = ap.parse_args()
    ctx = _native.context(0)
    mode = _native.GAUSS_ANGLESUM if a.mode == "anglesum" else _native.GAUSS_MODES[a.mode]
    if a.case == "kusari":
        m = gen.kusari_tube(after=True)
        from paper_2106_12655_b200.pls import upload
        upload(m, ctx)
        for _ in range(a.reps):
            device_step(ctx, m.xi, excluded_keys(()), DiscretizationParams(), mode=mode)
    else:
        if a.case == "torus":
            x, y = gen.torus_pair(2, 3, a.n)
        else:
            x, y = gen.ribbon_pair(10, a.n)
        for _ in range(a.reps):
            v = ctx.link_direct(x, y, mode)
        print("raw", v, "pairs", a.n * a.n)
    ctx.synchronize()


if __name__ == "__main__":
    main()
