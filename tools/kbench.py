"""Gauss-kernel A/B microbenchmark (CUDA events around the kernel only).

  python tools/kbench.py [--modes 0,16,17,18] [--reps 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2106_12655_b200 import _native, generators as gen  # noqa: E402


def bench_staged(ctx, modes, reps, label, sp):
    n = ctx.prepare_gauss()
    base = None
    for mode in modes:
        ts = []
        for _ in range(reps + 2):
            ctx.gauss_run(mode, 0, n)
            ts.append(ctx.gauss_event_ms())
        raw, lk, fl = ctx.gauss_reduce()
        if mode == 0:   # the fused path's pair-claiming kernel on the same pairs
            tp = []
            for _ in range(reps + 2):
                ctx.gauss_run_pairs(mode)
                tp.append(ctx.gauss_event_ms())
            print(f"{label:10s} pair kernel best {min(tp[2:]):8.3f} ms med {float(np.median(tp[2:])):8.3f} ms", flush=True)
        if base is None:
            base = raw
        best = min(ts[2:])
        med = float(np.median(ts[2:]))
        print(f"{label:10s} mode={mode} items={n} best {best:8.3f} ms med {med:8.3f} ms -> {sp / best / 1e-3:.3e} "
              f"seg-pairs/s  max|raw-raw0|={np.max(np.abs(raw - base)):.2e} lk={lk[:3]}", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="0")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-ribbon", action="store_true", help="skip the 100k x 100k ribbon pair (its pair-kernel run is ~20 s)")
    a = ap.parse_args()
    modes = [int(x) for x in a.modes.split(",")]
    ctx = _native.context(0)
    m = gen.kusari_tube(after=True)
    coeffs, t, off = m.packed()
    ctx.upload_model(coeffs, t, off)
    ctx.run_pipeline(None, m.xi, 2.220446049250313e-16, 64, 1 << 22)
    verts, voff = ctx.get_polylines()
    pairs = ctx.get_pairs()
    nv = np.diff(voff)
    sp = int(np.sum(nv[pairs[:, 0]] * nv[pairs[:, 1]]))
    bench_staged(ctx, modes, a.reps, "kusari", sp)
    for n in () if a.no_ribbon else (100_000,):
        x, y = gen.ribbon_pair(10, n)
        off2 = np.array([0, n, 2 * n], dtype=np.int64)
        ctx.stage_polylines(np.concatenate([x, y]), off2, np.array([[0, 1]], dtype=np.int32))
        bench_staged(ctx, modes, max(3, a.reps // 3), f"ribbon{n // 1000}k", n * n)
    e4 = gen.european_4in1(32, 32)
    c, t, o = e4.packed()
    ctx.upload_model(c, t, o)
    ctx.run_pipeline(None, e4.xi, 2.220446049250313e-16, 64, 1 << 22)
    verts, voff = ctx.get_polylines()
    pairs = ctx.get_pairs()
    nv = np.diff(voff)
    bench_staged(ctx, modes, a.reps, "e4in1", int(np.sum(nv[pairs[:, 0]] * nv[pairs[:, 1]])))


if __name__ == "__main__":
    main()
