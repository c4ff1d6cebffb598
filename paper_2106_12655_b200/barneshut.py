"""Barnes-Hut evaluation of the Gauss linking integral — drop-in for
linkcert.barneshut (barneshut.py:1-375), on the GPU.

Each loop gets a segment BVH with monopole / dipole / quadrupole moments (a
moment tree, built on the device: csrc/bh.cu, the reference's median split
and node numbering); a dual-tree traversal evaluates far-field node pairs with
the Taylor expansion of the Green's-function gradient and leaf pairs with the
exact arctangent term (breadth-first over node pairs, every level one kernel).
The running truncation estimate drives the reference's one-shot rerun with a
larger opening parameter.  Node boxes, moments, far-field terms and the
opening decisions are bitwise the reference's; only leaf-pair atan2 ulps and
the summation order differ (|delta| ~ 1e-15).

Batched use (certificates): `evaluate_pairs` runs every loop pair of a model
through one forest and two traversals instead of one tree pair at a time.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native

FOUR_PI = 4.0 * math.pi


@dataclass
class BarnesHutParams:
    """barneshut.py:25-41."""

    beta_init: float = 2.0
    beta_max: float = 10.0
    e_target: float = 0.2
    k_const: float = 1.0 / FOUR_PI
    order: str = "quadrupole"  # "dipole" or "quadrupole"
    adaptive: bool = True

    def __post_init__(self):
        if not (1.0 <= self.beta_init <= self.beta_max):
            raise ValueError("require 1 <= beta_init <= beta_max")
        if not self.e_target > 0.0:
            raise ValueError("e_target must be positive")
        if self.order not in ("dipole", "quadrupole"):
            raise ValueError(f"unknown expansion order {self.order!r}")


class _Bvh:
    """The fields of the reference's bvh.BvhTree a moment tree exposes (bvh.py:157-205)."""

    def __init__(self, nodes, prim_lo, prim_hi):
        self.node_lo, self.node_hi = nodes["node_lo"], nodes["node_hi"]
        self.left, self.right = nodes["left"], nodes["right"]
        self.start, self.end = nodes["start"], nodes["end"]
        self.prim_order = nodes["prim_order"]
        self.prim_lo, self.prim_hi = prim_lo, prim_hi

    @property
    def num_primitives(self):
        return self.prim_lo.shape[0]

    @property
    def num_nodes(self):
        return self.node_lo.shape[0]

    def depth(self):
        depths = {0: 1}
        best = 1
        for node in range(self.num_nodes):
            d = depths[node]
            best = max(best, d)
            if self.left[node] >= 0:
                depths[int(self.left[node])] = d + 1
                depths[int(self.right[node])] = d + 1
        return best


class MomentNode:
    """Read-only view of one node of a moment tree (barneshut.py:243-292)."""

    def __init__(self, tree, index):
        self._tree = tree
        self.index = index

    @property
    def box(self):
        from .geometry import Aabb

        t = self._tree.bvh
        return Aabb(t.node_lo[self.index], t.node_hi[self.index])

    @property
    def center(self):
        return self._tree.center[self.index]

    @property
    def radius(self):
        return float(self._tree.radius[self.index])

    @property
    def c_m(self):
        return self._tree.cm[self.index]

    @property
    def c_d(self):
        return self._tree.cd[self.index]

    @property
    def c_q(self):
        return self._tree.cq[self.index]

    @property
    def is_leaf(self):
        return self._tree.bvh.left[self.index] < 0

    def children(self):
        if self.is_leaf:
            return ()
        t = self._tree.bvh
        return (MomentNode(self._tree, int(t.left[self.index])), MomentNode(self._tree, int(t.right[self.index])))

    def segment(self):
        t = self._tree
        s = int(t.bvh.prim_order[int(t.bvh.start[self.index])])
        return t.seg_a[s], t.seg_b[s]


class MomentTree:
    """Segment BVH of one polyline loop with multipole moments per node
    (barneshut.py:295-323).  The tree lives on the device; node arrays are
    copied to the host on first access."""

    _HOST = ("center", "radius", "cm", "cd", "cq", "ncm", "ncd", "ncq")

    def __init__(self, loop):
        verts = loop.vertices if hasattr(loop, "vertices") else np.asarray(loop, float)
        self.seg_a = np.ascontiguousarray(verts)
        if self.seg_a.ndim != 2 or self.seg_a.shape[1:] != (3,) or self.seg_a.shape[0] == 0:
            raise ValueError("expected matching (m, 3) box corner arrays, m >= 1")
        # the device derives segment ends itself; seg_b / loop_length are host views made on first use
        self._forest = _native.context().bh_forest(self.seg_a, np.array([0, len(self.seg_a)], dtype=np.int64))
        self._nodes = None

    def _host(self):
        if self._nodes is None:
            self._nodes = self._forest.nodes()
        return self._nodes

    def __getattr__(self, name):
        if name in MomentTree._HOST:
            return self._host()[name]
        if name == "seg_b":
            self.__dict__["seg_b"] = np.ascontiguousarray(np.roll(self.seg_a, -1, axis=0))
            return self.seg_b
        if name == "loop_length":
            self.__dict__["loop_length"] = float(np.sum(np.linalg.norm(self.seg_b - self.seg_a, axis=1)))
            return self.loop_length
        if name == "bvh":
            lo = np.minimum(self.seg_a, self.seg_b)
            hi = np.maximum(self.seg_a, self.seg_b)
            bvh = _Bvh(self._host(), lo, hi)
            self.__dict__["bvh"] = bvh
            return bvh
        raise AttributeError(name)

    @property
    def root(self):
        return MomentNode(self, 0)


def build_moment_tree(loop) -> MomentTree:
    return MomentTree(loop)


def far_field_eval(node1: MomentNode, node2: MomentNode, order="quadrupole") -> float:
    """Far-field expansion for one node pair (monopole+dipole[+quadrupole]) (barneshut.py:330-345)."""
    f1, f2 = node1._tree._forest, node2._tree._forest
    return float(f1.far_field(node1.index, f2, node2.index, order == "quadrupole"))


@dataclass
class BarnesHutResult:
    value: float
    e_estimate: float
    beta_used: float
    reran: bool


def _dual_eval(tree1, tree2, beta, quadrupole, k_const):
    lam, est, _ = tree1._forest.eval(tree2._forest, [[0, 0]], beta, quadrupole, k_const)
    return float(lam[0]), float(est[0])


def barnes_hut_detailed(tree1: MomentTree, tree2: MomentTree, params=None) -> BarnesHutResult:
    """barneshut.py:355-371."""
    params = params or BarnesHutParams()
    quad = params.order == "quadrupole"
    lam, e_est = _dual_eval(tree1, tree2, params.beta_init, quad, params.k_const)
    beta_used = params.beta_init
    reran = False
    if params.adaptive:
        beta_t = (e_est / params.e_target) ** 0.25 * params.beta_init
        if beta_t > params.beta_init:
            beta_used = min(beta_t, params.beta_max)
            lam, _ = _dual_eval(tree1, tree2, beta_used, quad, params.k_const)
            reran = True
    return BarnesHutResult(float(lam), float(e_est), float(beta_used), reran)


def link_barnes_hut(tree1: MomentTree, tree2: MomentTree, params=None) -> float:
    return barnes_hut_detailed(tree1, tree2, params).value


def evaluate_pairs(polylines, pairs, params=None):
    """Barnes-Hut for many loop pairs at once: one moment forest over the loops
    the pairs use, one batched traversal at beta_init, one for the pairs the
    adaptive rule reruns (each with its own beta, computed as the reference's
    barnes_hut_detailed does per pair).  Returns (value, e_estimate, beta_used,
    reran) arrays in pair order."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    if pairs.shape[0] == 0:
        return evaluate_pairs_packed(np.zeros((0, 3)), np.zeros(1, dtype=np.int64), pairs, params)
    used, tree_of = np.unique(pairs, return_inverse=True)
    blocks = [np.asarray(polylines[int(i)].vertices if hasattr(polylines[int(i)], "vertices")
                         else polylines[int(i)], dtype=np.float64) for i in used]
    off = np.zeros(len(blocks) + 1, dtype=np.int64)
    np.cumsum([len(b) for b in blocks], out=off[1:])
    return evaluate_pairs_packed(np.concatenate(blocks), off, tree_of.reshape(-1, 2), params)


def evaluate_pairs_packed(verts, loop_off, pairs, params=None):
    """evaluate_pairs on packed loops: verts (M, 3), loop t = rows
    [loop_off[t], loop_off[t+1]); pairs index the loops."""
    params = params or BarnesHutParams()
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    P = pairs.shape[0]
    value = np.zeros(P)
    est = np.zeros(P)
    beta_used = np.full(P, float(params.beta_init))
    reran = np.zeros(P, dtype=bool)
    if P == 0:
        return value, est, beta_used, reran
    tree_pairs = pairs.astype(np.int32)
    forest = _native.context().bh_forest(verts, loop_off)
    quad = params.order == "quadrupole"
    value, est, _ = forest.eval(forest, tree_pairs, params.beta_init, quad, params.k_const)
    if params.adaptive:
        redo, betas = [], []
        for k, e in enumerate(est.tolist()):   # Python float arithmetic, as barneshut.py:364
            beta_t = (e / params.e_target) ** 0.25 * params.beta_init
            if beta_t > params.beta_init:
                redo.append(k)
                betas.append(min(beta_t, params.beta_max))
        if redo:
            lam2, _, _ = forest.eval(forest, tree_pairs[redo], np.asarray(betas), quad, params.k_const)
            value[redo] = lam2
            beta_used[redo] = betas
            reran[redo] = True
    return value, est, beta_used, reran
