"""Scratch GPU probe: FP64 peak, Gauss-sum parity vs the C oracle, throughput.

Run on the GPU box:  python tools/gpu_probe.py
"""
import ctypes
import math
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2106_12655_b200 import _native as nat  # noqa: E402

ORC = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "..", "oracle", "liboracle_gauss.so"))
ORC.oracle_link_atan.restype = ctypes.c_double
ORC.oracle_evaluate_pairs.restype = ctypes.c_int
ORC.oracle_link_atan_rows.restype = ctypes.c_double
DP = ctypes.POINTER(ctypes.c_double)


def closed(v):
    return np.ascontiguousarray(np.vstack([v, v[:1]]))


def oracle_link(a, b):
    l, k = closed(a), closed(b)
    return ORC.oracle_link_atan(l.ctypes.data_as(DP), len(a), k.ctypes.data_as(DP), len(b))


def torus_pair(T, P, n, R=2.0, r=0.5):
    t = np.linspace(0.0, 1.0, n, endpoint=False)
    ang = 2.0 * math.pi * T * t
    core = np.stack([R * np.cos(ang), R * np.sin(ang), np.zeros(n)], axis=1)
    tor = 2.0 * math.pi * t
    pol = 2.0 * math.pi * P * t
    rad = R + r * np.cos(pol)
    w = np.stack([rad * np.cos(tor), rad * np.sin(tor), -r * np.sin(pol)], axis=1)
    return core, w


def ribbon(lam, n, ax=10.0, tr=1.0):
    t = np.linspace(0.0, 1.0, n, endpoint=False)
    tor = 2.0 * math.pi * t
    tw = 2.0 * math.pi * lam * t
    out = []
    for ph in (0.0, math.pi):
        rad = ax + tr * np.cos(tw + ph)
        out.append(np.stack([rad * np.cos(tor), rad * np.sin(tor), -tr * np.sin(tw + ph)], axis=1))
    return out


def circle(n, c, u, v, r=1.0):
    t = np.linspace(0.0, 2.0 * math.pi, n, endpoint=False)
    return np.asarray(c, float) + r * np.outer(np.cos(t), u) + r * np.outer(np.sin(t), v)


def main():
    ctx = nat.context(0)
    fl, ms = ctx.probe_fp64_peak()
    print(f"FP64 DFMA peak: {fl/1e12:.2f} TFLOP/s ({ms:.1f} ms)", flush=True)

    # --- parity on C1 --------------------------------------------------------
    for (T, P) in [(1, 1), (1, 2), (1, 3), (1, 5), (2, 3), (3, 5), (10, 10)]:
        a, b = torus_pair(T, P, 1024)
        o = oracle_link(a, b)
        vals = [ctx.link_direct(a, b, m) for m in (0, 1, 2)]
        print(f"torus({T},{P}) oracle={o!r} phase={vals[0]!r} atan={vals[1]!r} ref={vals[2]!r} "
              f"maxdiff={max(abs(v - o) for v in vals):.2e}", flush=True)
    ex, ey, ez = np.eye(3)
    a = circle(1024, (0, 0, 0), ex, ey)
    b = circle(1024, (1, 0, 0), ez, ex)
    print("hopf", oracle_link(a, b), [ctx.link_direct(a, b, m) for m in (0, 1, 2)])
    a = circle(48, (0, 0, 0), ex, ey)
    b = circle(48, (5, 0, 0), ex, ey)
    print("coplanar", oracle_link(a, b), [ctx.link_direct(a, b, m) for m in (0, 1, 2)])
    rng = np.random.default_rng(0)
    for trial in range(3):
        a = rng.normal(size=(37 + trial * 50, 3))
        b = rng.normal(size=(53 + trial * 30, 3)) + 0.3
        o = oracle_link(a, b)
        vals = [ctx.link_direct(a, b, m) for m in (0, 1, 2)]
        print(f"random{trial} oracle={o!r} diffs={[abs(v - o) for v in vals]}", flush=True)

    # --- chainmail-like batch: 18752 pairs of 64x64 --------------------------
    P = 18752
    rings = []
    pairs = []
    for k in range(P):
        c = np.array([3.0 * (k % 137), 3.0 * (k // 137), 0.0])
        rings.append(circle(64, c, ex, ey))
        rings.append(circle(64, c + [1.0, 0, 0], ez, ex))
        pairs.append((2 * k, 2 * k + 1))
    verts = np.concatenate(rings)
    off = np.arange(0, 64 * len(rings) + 1, 64, dtype=np.int64)
    pairs = np.array(pairs, dtype=np.int32)
    for mode in (0, 1, 2):
        raw, lk, flags = ctx.evaluate_pairs(verts, off, pairs, mode)
        best = 1e9
        for _ in range(5):
            ctx.evaluate_pairs(verts, off, pairs, mode)
            best = min(best, ctx.last_gauss_ms())
        sp = P * 64 * 64
        print(f"chainmail-like mode={mode} kernel {best:.3f} ms -> {sp/best/1e-3:.3e} seg-pairs/s; "
              f"lk all 1: {bool(np.all(lk == 1))} max|raw-1|={np.max(np.abs(raw-1)):.2e}", flush=True)
    # oracle on a sample of pairs
    raw_o = np.empty(200)
    ORC.oracle_evaluate_pairs(verts.ctypes.data_as(DP), off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                              pairs.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), ctypes.c_int64(200), 0,
                              os.cpu_count(), raw_o.ctypes.data_as(DP))
    raw, lk, flags = ctx.evaluate_pairs(verts, off, pairs, 0)
    print("chainmail oracle maxdiff (200 pairs):", np.max(np.abs(raw[:200] - raw_o)))

    # --- big pair: ribbon --------------------------------------------------------
    for n in (20000, 100000):
        a, b = ribbon(10, n)
        for mode in (0, 1, 2):
            if mode == 2 and n > 20000:
                continue
            v = ctx.link_direct(a, b, mode)
            t0 = time.perf_counter()
            v = ctx.link_direct(a, b, mode)
            ms = ctx.last_gauss_ms()
            print(f"ribbon n={n} mode={mode} raw={v!r} err={abs(v-10):.2e} kernel {ms:.2f} ms "
                  f"-> {n*n/ms/1e-3:.3e} seg-pairs/s (wall {time.perf_counter()-t0:.3f}s)", flush=True)
        if n == 20000:
            t0 = time.perf_counter()
            l, k = closed(a), closed(b)
            o = ORC.oracle_link_atan_rows(l.ctypes.data_as(DP), ctypes.c_int64(n), k.ctypes.data_as(DP),
                                          ctypes.c_int64(0), ctypes.c_int64(n), os.cpu_count())
            print(f"oracle ribbon {n}: {o!r} in {time.perf_counter()-t0:.2f}s on {os.cpu_count()} threads")


if __name__ == "__main__":
    main()
