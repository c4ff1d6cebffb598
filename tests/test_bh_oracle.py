"""Pin the Barnes-Hut CPU oracle (oracle/bh_oracle.py) against vectors produced
by the reference itself (tests/golden/bh_golden.*, make_golden_bh.py).  CPU only.

The oracle restates bvh._build / barneshut._compute_moments / _far_field /
_dual_eval in IEEE double without contraction, like the numba kernels
(fastmath off): trees, moments and far-field values must be BITWISE equal,
and Barnes-Hut sums too (same depth-first summation order, same libm atan2).
"""

import numpy as np
import pytest

import paper_2106_12655_b200 as lc

TREE = ("node_lo", "node_hi", "left", "right", "start", "end", "prim_order")
MOM = ("center", "radius", "cm", "cd", "cq", "ncm", "ncd", "ncq")
SMALL_BH = ("hopf32", "arcs_far", "torus23_beta1e6", "wobbly_hopf", "self_pair")


def _trees(bh_golden):
    return bh_golden["trees"]


@pytest.mark.parametrize("name", ["circle16", "noisy64", "circle33", "circle50", "ties24", "single3", "helix300",
                                  "random400"])
def test_oracle_tree_and_moments_bitwise(bh_oracle, bh_arrays, name):
    t = bh_oracle.Tree(bh_arrays[f"tree_{name}_verts"])
    for f in TREE:
        assert np.array_equal(getattr(t, f), bh_arrays[f"tree_{name}_{f}"]), f
    for f in MOM:
        assert np.array_equal(getattr(t, f), bh_arrays[f"tree_{name}_{f}"]), f


def test_oracle_far_field_bitwise(bh_oracle, bh_arrays):
    vals = bh_arrays["ff_values"]
    trees = {}
    for dist, na, nb, quad, want in vals:
        key = int(dist)
        if key not in trees:
            trees[key] = (bh_oracle.Tree(bh_arrays[f"ff_{key}_a"]), bh_oracle.Tree(bh_arrays[f"ff_{key}_b"]))
        a, b = trees[key]
        na, nb = int(na), int(nb)
        got = bh_oracle.far_field(b.center[nb] - a.center[na], a.cm[na], a.cd[na], a.cq[na], b.cm[nb], b.cd[nb],
                                  b.cq[nb], bool(quad))
        assert got == want, (dist, na, nb, quad)


@pytest.mark.parametrize("name", SMALL_BH)
def test_oracle_barnes_hut_bitwise(bh_oracle, bh_golden, bh_arrays, name):
    g = next(c for c in bh_golden["bh"] if c["name"] == name)
    p = lc.BarnesHutParams(**g["params"])
    a, b = bh_oracle.Tree(bh_arrays[f"bh_{name}_a"]), bh_oracle.Tree(bh_arrays[f"bh_{name}_b"])
    value, est, beta, reran = bh_oracle.barnes_hut(a, b, p.beta_init, p.beta_max, p.e_target, p.k_const, p.order,
                                                   p.adaptive)
    assert (value, est, beta, reran) == (g["value"], g["e_estimate"], g["beta_used"], g["reran"])


def test_params_validation():
    """test_barneshut.py:141-149."""
    with pytest.raises(ValueError):
        lc.BarnesHutParams(beta_init=0.5)
    with pytest.raises(ValueError):
        lc.BarnesHutParams(beta_init=5.0, beta_max=2.0)
    with pytest.raises(ValueError):
        lc.BarnesHutParams(e_target=0.0)
    with pytest.raises(ValueError):
        lc.BarnesHutParams(order="octupole")
    assert lc.KernelChoice(method="bh").tag == "bh:quadrupole"
    assert lc.KernelChoice(method="bh", bh=lc.BarnesHutParams(order="dipole")).tag == "bh:dipole"
