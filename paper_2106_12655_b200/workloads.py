"""Vertex arrays of the benchmark workloads (BASELINE.json configs[1..4];
SURVEY.md Appendix B) — numpy only.

This module imports nothing from the package (no ctypes, no library), so the
CPU reference arm of bench.py can build exactly the same inputs by loading
this file alone; paper_2106_12655_b200.generators wraps the arrays into
CurveModels (CurveModel.from_polyline_arrays).  Every builder returns
(verts (V, 3) float64, loop_off (L+1) int64) of closed polylines.
"""

from __future__ import annotations

import math

import numpy as np


def ring(n, center, u, v, radius=1.0):
    """center + r cos(t) u + r sin(t) v at t = 2 pi k / n (generators.py:27-33 expression order)."""
    t = np.linspace(0.0, 2.0 * math.pi, n, endpoint=False)
    return (np.asarray(center, dtype=float) + radius * np.outer(np.cos(t), u)
            + radius * np.outer(np.sin(t), v))


def rings(n, centers, us, vs, radii):
    """Many rings at once; elementwise identical to `ring` for each row."""
    t = np.linspace(0.0, 2.0 * math.pi, n, endpoint=False)
    c, s = np.cos(t)[None, :, None], np.sin(t)[None, :, None]
    radii = np.asarray(radii, dtype=float).reshape(-1, 1, 1)
    return (np.asarray(centers, float)[:, None, :] + radii * (c * np.asarray(us, float)[:, None, :])
            + radii * (s * np.asarray(vs, float)[:, None, :]))


def _packed(vert_blocks):
    """(R, n, 3) ring block(s) -> (verts (V, 3), loop_off (L+1))."""
    verts = np.concatenate([b.reshape(-1, 3) for b in vert_blocks])
    counts = np.concatenate([np.full(b.shape[0], b.shape[1], dtype=np.int64) for b in vert_blocks])
    off = np.zeros(len(counts) + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return verts, off


def european_4in1_params(rows=32, cols=32, pitch=1.4, row_pitch=1.2, tilt=0.6):
    """Centres / planes of the European 4-in-1 sheet (Appendix B.1); ring = row*cols + col."""
    r, c = np.divmod(np.arange(rows * cols), cols)
    centers = np.stack([c * pitch + (r % 2) * (0.5 * pitch), r * row_pitch, np.zeros(rows * cols)], axis=1)
    theta = np.where(r % 2 == 0, tilt, -tilt)
    us = np.stack([np.cos(theta), np.zeros_like(theta), np.sin(theta)], axis=1)
    vs = np.tile([0.0, 1.0, 0.0], (rows * cols, 1))
    return centers, us, vs


def european_4in1_vertices(rows=32, cols=32, n=64, radius=1.0, moved=None):
    """Config C2: European 4-in-1 chainmail sheet, `rows` x `cols` rings of n segments.

    `moved` = {ring index: new centre z} pulls rings out of the sheet (the
    Appendix B.1 pull-out edit moves ring 165 to z = 3).
    """
    centers, us, vs = european_4in1_params(rows, cols)
    if moved:
        for idx, z in moved.items():
            centers[idx, 2] = z
    return _packed([rings(n, centers, us, vs, np.full(len(centers), radius))])


def kusari_tube_params(n_around=95, rows=49, partial=81, pitch=2.2, big_radius=1.0, small_radius=0.6):
    """Ring table of the Japanese 4-in-1 tube (Appendix B.2).

    Returns (centers, us, vs, radii, conn) where conn lists, for every
    connector ring, (kind, r, c) with kind 0 = around (between (r,c) and
    (r,c+1)), 1 = along (between (r,c) and (r+1,c)).
    """
    Rc = n_around * pitch / (2.0 * math.pi)
    ez = np.array([0.0, 0.0, 1.0])

    def e_r(phi):
        return np.array([math.cos(phi), math.sin(phi), 0.0])

    def e_phi(phi):
        return np.array([-math.sin(phi), math.cos(phi), 0.0])

    present = [(r, c) for r in range(rows) for c in range(n_around)] + [(rows, c) for c in range(partial)]
    pset = set(present)
    centers, us, vs, radii, conn = [], [], [], [], []
    for r, c in present:
        phi = 2.0 * math.pi * c / n_around
        centers.append(Rc * e_r(phi) + r * pitch * ez)
        us.append(e_phi(phi))
        vs.append(ez)
        radii.append(big_radius)
    for r, c in present:
        if (r, (c + 1) % n_around) in pset:
            phi = 2.0 * math.pi * (c + 0.5) / n_around
            centers.append(Rc * math.cos(math.pi / n_around) * e_r(phi) + r * pitch * ez)
            us.append(e_phi(phi))
            vs.append(e_r(phi))
            radii.append(small_radius)
            conn.append((0, r, c))
        if (r + 1, c) in pset:
            phi = 2.0 * math.pi * c / n_around
            centers.append(Rc * e_r(phi) + (r + 0.5) * pitch * ez)
            us.append(ez)
            vs.append(e_r(phi))
            radii.append(small_radius)
            conn.append((1, r, c))
    return (np.array(centers), np.array(us), np.array(vs), np.array(radii), conn, Rc)


def kusari_tube_vertices(n=64, after=False, **kw):
    """Config C3: Kusari-scale chainmail tube — 14,112 rings / 18,752 links at the defaults.

    after=True applies the Appendix B.2 edits: connector 100 moved by
    (0, 0, 500); connector 2000 replaced by an around-connector at the
    dangling edge (row 49, c + 1/2 = 80.5); connector 5000 reversed.
    """
    centers, us, vs, radii, conn, Rc = kusari_tube_params(**kw)
    n_big = len(centers) - len(conn)
    block = rings(n, centers, us, vs, radii)
    if after:
        n_around = kw.get("n_around", 95)
        pitch = kw.get("pitch", 2.2)
        rows = kw.get("rows", 49)
        block = block.copy()
        block[n_big + 100] += np.array([0.0, 0.0, 500.0])
        phi = 2.0 * math.pi * (kw.get("partial", 81) - 1 + 0.5) / n_around
        er = np.array([math.cos(phi), math.sin(phi), 0.0])
        ephi = np.array([-math.sin(phi), math.cos(phi), 0.0])
        c2000 = Rc * math.cos(math.pi / n_around) * er + rows * pitch * np.array([0.0, 0.0, 1.0])
        block[n_big + 2000] = ring(n, c2000, ephi, er, radii[n_big + 2000])
        block[n_big + 5000] = block[n_big + 5000][::-1].copy()
    return _packed([block])


def knit_course(k, n, W=100, h=1.0, A=0.9, B=0.3):
    """Course k of the interlocking-course knit tube (Appendix B.3)."""
    R = W * 1.5 / (2.0 * math.pi)
    s = 2.0 * math.pi * np.arange(n) / n
    sign = -1.0 if k % 2 else 1.0
    z = k * h + sign * A * np.sin(W * s)
    rho = R + sign * B * np.cos(W * s)
    return np.stack([rho * np.cos(s), rho * np.sin(s), z], axis=1)


def knit_tube_vertices(courses=200, n=100_000, W=100):
    """Config C4: `courses` closed courses of n segments; adjacent courses link -W times."""
    return _packed([np.stack([knit_course(k, n, W) for k in range(courses)])])
