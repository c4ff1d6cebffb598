"""TEST INFRASTRUCTURE ONLY — CPU oracle for the Barnes-Hut path.

Only tests/ may import this module; the product package never does.

A pure-Python restatement (IEEE double, no FMA: the numba kernels run with
fastmath off) of:
  build_tree     <- linkcert/bvh.py:17-90 (_build, leaf_size 1)
  moments        <- linkcert/barneshut.py:43-90 (_compute_moments), :93-112 (_norms)
  far_field      <- linkcert/barneshut.py:120-172 (_far_field)
  dual_eval      <- linkcert/barneshut.py:175-240 (_dual_eval, depth-first stack)
  pair_lambda    <- linkcert/direct.py:19-46 (_pair_lambda)
  barnes_hut     <- linkcert/barneshut.py:355-371 (barnes_hut_detailed)
For small loops only (pure-Python loops).  Pinned against vectors produced by
the reference itself: tests/golden/bh_golden.npz (tests/golden/make_golden_bh.py)
in tests/test_bh_oracle.py.
"""

from __future__ import annotations

import math

import numpy as np

FOUR_PI = 4.0 * math.pi
TWO_PI = 2.0 * math.pi


def build_tree(lo, hi):
    """bvh._build with leaf_size=1: node_lo, node_hi, left, right, start, end, order."""
    m = lo.shape[0]
    centers = 0.5 * (lo + hi)
    n_max = 2 * m - 1
    node_lo = np.empty((n_max, 3))
    node_hi = np.empty((n_max, 3))
    left = np.full(n_max, -1, dtype=np.int64)
    right = np.full(n_max, -1, dtype=np.int64)
    start = np.zeros(n_max, dtype=np.int64)
    end = np.zeros(n_max, dtype=np.int64)
    order = np.arange(m)
    n_nodes = 1
    stack = [(0, 0, m)]
    while stack:
        node, s, e = stack.pop()
        blo = lo[order[s]].copy()
        bhi = hi[order[s]].copy()
        for k in range(s + 1, e):
            p = order[k]
            for d in range(3):
                if lo[p, d] < blo[d]:
                    blo[d] = lo[p, d]
                if hi[p, d] > bhi[d]:
                    bhi[d] = hi[p, d]
        node_lo[node], node_hi[node] = blo, bhi
        start[node], end[node] = s, e
        if e - s <= 1:
            continue
        axis, best = 0, bhi[0] - blo[0]
        for d in (1, 2):
            w = bhi[d] - blo[d]
            if w > best:
                best, axis = w, d
        idx = np.sort(order[s:e])
        order[s:e] = idx[np.argsort(centers[idx, axis], kind="mergesort")]
        mid = s + (e - s) // 2
        lc, rc = n_nodes, n_nodes + 1
        n_nodes += 2
        left[node], right[node] = lc, rc
        stack.append((lc, s, mid))
        stack.append((rc, mid, e))
    return node_lo, node_hi, left, right, start, end, order


def moments(node_lo, node_hi, left, right, start, order, seg_a, seg_b):
    """_compute_moments + _norms: center, radius, cm, cd, cq, ncm, ncd, ncq."""
    n = node_lo.shape[0]
    center = 0.5 * (node_lo + node_hi)
    radius = np.empty(n)
    for v in range(n):
        dx, dy, dz = (float(node_hi[v, k] - node_lo[v, k]) for k in range(3))
        radius[v] = 0.5 * math.sqrt(dx * dx + dy * dy + dz * dz)
    cm = np.zeros((n, 3))
    cd = np.zeros((n, 3, 3))
    cq = np.zeros((n, 3, 3, 3))
    for v in range(n - 1, -1, -1):
        if left[v] < 0:
            s = order[start[v]]
            mid = 0.5 * (seg_a[s] + seg_b[s])
            d = seg_b[s] - seg_a[s]
            cm[v] = d
            rloc = mid - center[v]
            for i in range(3):
                for j in range(3):
                    cd[v, i, j] = d[i] * rloc[j]
                    for k in range(3):
                        cq[v, i, j, k] = d[i] * (d[j] * d[k] / 12.0 + rloc[j] * rloc[k])
        else:
            for c in (left[v], right[v]):
                rc = center[c] - center[v]
                for i in range(3):
                    cm[v, i] += cm[c, i]
                    for j in range(3):
                        cd[v, i, j] += cd[c, i, j] + cm[c, i] * rc[j]
                        for k in range(3):
                            cq[v, i, j, k] += (cq[c, i, j, k] + cd[c, i, j] * rc[k] + cd[c, i, k] * rc[j]
                                               + cm[c, i] * rc[j] * rc[k])
    ncm, ncd, ncq = np.empty(n), np.empty(n), np.empty(n)
    for v in range(n):
        ncm[v] = math.sqrt(cm[v, 0] * cm[v, 0] + cm[v, 1] * cm[v, 1] + cm[v, 2] * cm[v, 2])
        s2 = 0.0
        for i in range(3):
            for j in range(3):
                s2 += cd[v, i, j] * cd[v, i, j]
        ncd[v] = math.sqrt(s2)
        s3 = 0.0
        for i in range(3):
            for j in range(3):
                for k in range(3):
                    s3 += cq[v, i, j, k] * cq[v, i, j, k]
        ncq[v] = math.sqrt(s3)
    return center, radius, cm, cd, cq, ncm, ncd, ncq


class Tree:
    """MomentTree (barneshut.py:298-312) on the host."""

    def __init__(self, verts):
        verts = np.asarray(verts, dtype=np.float64)
        self.seg_a = np.ascontiguousarray(verts)
        self.seg_b = np.ascontiguousarray(np.roll(verts, -1, axis=0))
        lo = np.minimum(self.seg_a, self.seg_b)
        hi = np.maximum(self.seg_a, self.seg_b)
        (self.node_lo, self.node_hi, self.left, self.right, self.start, self.end,
         self.prim_order) = build_tree(lo, hi)
        (self.center, self.radius, self.cm, self.cd, self.cq, self.ncm, self.ncd,
         self.ncq) = moments(self.node_lo, self.node_hi, self.left, self.right, self.start, self.prim_order,
                             self.seg_a, self.seg_b)


def _cross(ax, ay, az, bx, by, bz):
    return ay * bz - az * by, az * bx - ax * bz, ax * by - ay * bx


def far_field(r, cm1, cd1, cq1, cm2, cd2, cq2, quadrupole):
    rx, ry, rz = (float(x) for x in r)
    cm1, cm2 = [float(x) for x in cm1], [float(x) for x in cm2]
    r2 = rx * rx + ry * ry + rz * rz
    rn = math.sqrt(r2)
    inv3 = 1.0 / (FOUR_PI * r2 * rn)
    inv5 = inv3 / r2
    inv7 = inv5 / r2
    rr = (rx, ry, rz)
    wx, wy, wz = _cross(*cm1, *cm2)
    total = -(wx * rx + wy * ry + wz * rz) * inv3
    for b in range(3):
        u1 = _cross(float(cd1[0, b]), float(cd1[1, b]), float(cd1[2, b]), *cm2)
        u2 = _cross(*cm1, float(cd2[0, b]), float(cd2[1, b]), float(cd2[2, b]))
        vx, vy, vz = u2[0] - u1[0], u2[1] - u1[1], u2[2] - u1[2]
        rb = rr[b]
        dot_vr = vx * rx + vy * ry + vz * rz
        hv = vx * (1.0 if b == 0 else 0.0) + vy * (1.0 if b == 1 else 0.0) + vz * (1.0 if b == 2 else 0.0)
        total -= (hv * r2 - 3.0 * dot_vr * rb) * inv5
    if quadrupole:
        for b in range(3):
            for c in range(3):
                q1 = _cross(float(cq1[0, b, c]), float(cq1[1, b, c]), float(cq1[2, b, c]), *cm2)
                q2 = _cross(*cm1, float(cq2[0, b, c]), float(cq2[1, b, c]), float(cq2[2, b, c]))
                dd = _cross(float(cd1[0, b]), float(cd1[1, b]), float(cd1[2, b]),
                            float(cd2[0, c]), float(cd2[1, c]), float(cd2[2, c]))
                vx = q1[0] + q2[0] - 2.0 * dd[0]
                vy = q1[1] + q2[1] - 2.0 * dd[1]
                vz = q1[2] + q2[2] - 2.0 * dd[2]
                rb, rc = rr[b], rr[c]
                dot_vr = vx * rx + vy * ry + vz * rz
                t = 0.0
                if b == c:
                    t += -3.0 * dot_vr * inv5
                t += -3.0 * (vx if b == 0 else (vy if b == 1 else vz)) * rc * inv5
                t += -3.0 * (vx if c == 0 else (vy if c == 1 else vz)) * rb * inv5
                t += 15.0 * dot_vr * rb * rc * inv7
                total -= 0.5 * t
    return total


def pair_lambda(l_j, l_j1, k_i, k_i1):
    ljx, ljy, ljz = (float(x) for x in l_j)
    lj1x, lj1y, lj1z = (float(x) for x in l_j1)
    kix, kiy, kiz = (float(x) for x in k_i)
    ki1x, ki1y, ki1z = (float(x) for x in k_i1)
    ax, ay, az = ljx - kix, ljy - kiy, ljz - kiz
    bx, by, bz = ljx - ki1x, ljy - ki1y, ljz - ki1z
    cx, cy, cz = lj1x - ki1x, lj1y - ki1y, lj1z - ki1z
    dx, dy, dz = lj1x - kix, lj1y - kiy, lj1z - kiz
    an = math.sqrt(ax * ax + ay * ay + az * az)
    bn = math.sqrt(bx * bx + by * by + bz * bz)
    cn = math.sqrt(cx * cx + cy * cy + cz * cz)
    dn = math.sqrt(dx * dx + dy * dy + dz * dz)
    p = ax * (by * cz - bz * cy) + ay * (bz * cx - bx * cz) + az * (bx * cy - by * cx)
    ab = ax * bx + ay * by + az * bz
    bc = bx * cx + by * cy + bz * cz
    ca = cx * ax + cy * ay + cz * az
    ad = ax * dx + ay * dy + az * dz
    dc = dx * cx + dy * cy + dz * cz
    d1 = an * bn * cn + ab * cn + bc * an + ca * bn
    d2 = an * dn * cn + ad * cn + dc * an + ca * dn
    return (math.atan2(p, d1) + math.atan2(p, d2)) / TWO_PI


def dual_eval(a: Tree, b: Tree, beta, quadrupole=True, k_const=1.0 / FOUR_PI):
    """_dual_eval: (lam, e_est, n_far, n_leaf) in the reference's depth-first order."""
    lam = 0.0
    e_est = 0.0
    n_far = n_leaf = 0
    stack = [(0, 0)]
    while stack:
        na, nb = stack.pop()
        rx, ry, rz = (float(b.center[nb, k] - a.center[na, k]) for k in range(3))
        dist = math.sqrt(rx * rx + ry * ry + rz * rz)
        ra, rb = float(a.radius[na]), float(b.radius[nb])
        if dist > beta * (ra + rb):
            lam += far_field((rx, ry, rz), a.cm[na], a.cd[na], a.cq[na], b.cm[nb], b.cd[nb], b.cq[nb], quadrupole)
            inv5 = 1.0 / (dist * ((dist * dist) * (dist * dist)))
            e_est += k_const * inv5 * (ra * float(b.ncm[nb]) * float(a.ncq[na])
                                       + rb * float(a.ncm[na]) * float(b.ncq[nb])
                                       + 3.0 * (float(a.ncd[na]) * float(b.ncq[nb]) + float(a.ncq[na]) * float(b.ncd[nb])))
            n_far += 1
            continue
        a_leaf, b_leaf = a.left[na] < 0, b.left[nb] < 0
        if a_leaf and b_leaf:
            sa = a.prim_order[a.start[na]]
            sb = b.prim_order[b.start[nb]]
            lam += pair_lambda(a.seg_a[sa], a.seg_b[sa], b.seg_a[sb], b.seg_b[sb])
            n_leaf += 1
            continue
        if not a_leaf and (b_leaf or ra > rb):
            stack.append((int(a.left[na]), nb))
            stack.append((int(a.right[na]), nb))
        else:
            stack.append((na, int(b.left[nb])))
            stack.append((na, int(b.right[nb])))
    return lam, e_est, n_far, n_leaf


def barnes_hut(a: Tree, b: Tree, beta_init=2.0, beta_max=10.0, e_target=0.2, k_const=1.0 / FOUR_PI,
               order="quadrupole", adaptive=True):
    """barnes_hut_detailed: (value, e_estimate, beta_used, reran)."""
    quad = order == "quadrupole"
    lam, e_est, _, _ = dual_eval(a, b, beta_init, quad, k_const)
    beta_used, reran = beta_init, False
    if adaptive:
        beta_t = (e_est / e_target) ** 0.25 * beta_init
        if beta_t > beta_init:
            beta_used = min(beta_t, beta_max)
            lam, _, _, _ = dual_eval(a, b, beta_used, quad, k_const)
            reran = True
    return float(lam), float(e_est), float(beta_used), reran
