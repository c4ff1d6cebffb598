"""Barnes-Hut on the GPU (csrc/bh.cu via lc_bh_*) against the reference's own
vectors (tests/golden/bh_golden.*) and the pinned oracle (oracle/bh_oracle.py),
plus the reference's test_barneshut.py behaviour.

Bar: tree topology, node boxes, moments and far-field terms BITWISE (bh.cu is
compiled without FMA contraction in the reference's operation order);
Barnes-Hut sums within 1e-12 (leaf atan2 ulps, breadth-first summation order);
the adaptive rerun decision, beta_used and integer certificates exact.
"""

import math

import numpy as np
import pytest

import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import barneshut, _native
from paper_2106_12655_b200.barneshut import MomentNode

pytestmark = pytest.mark.gpu

TREE = ("node_lo", "node_hi", "left", "right", "start", "end", "prim_order")
MOM = ("center", "radius", "cm", "cd", "cq", "ncm", "ncd", "ncq")
TREES = ["circle16", "noisy64", "circle33", "circle50", "ties24", "single3", "helix300", "random400"]


def _circle(n, center=(0.0, 0.0, 0.0), u=(1.0, 0.0, 0.0), v=(0.0, 1.0, 0.0), radius=1.0):
    t = np.linspace(0.0, 2.0 * math.pi, n, endpoint=False)
    return (np.asarray(center, dtype=float) + radius * np.outer(np.cos(t), np.asarray(u, dtype=float))
            + radius * np.outer(np.sin(t), np.asarray(v, dtype=float)))


@pytest.mark.parametrize("name", TREES)
def test_tree_and_moments_bitwise(gpu, bh_arrays, name):
    t = lc.build_moment_tree(bh_arrays[f"tree_{name}_verts"])
    for f in TREE:
        assert np.array_equal(getattr(t.bvh, f), bh_arrays[f"tree_{name}_{f}"]), f
    for f in MOM:
        assert np.array_equal(getattr(t, f), bh_arrays[f"tree_{name}_{f}"]), f
    assert t.loop_length == bh_arrays[f"tree_{name}_loop_length"][0]


def test_forest_equals_single_trees(gpu, bh_arrays):
    """One forest of many loops = the loops' trees one by one (per-tree numbering)."""
    blocks = [bh_arrays[f"tree_{n}_verts"] for n in TREES]
    off = np.zeros(len(blocks) + 1, dtype=np.int64)
    np.cumsum([len(b) for b in blocks], out=off[1:])
    nodes = gpu.bh_forest(np.concatenate(blocks), off).nodes()
    noff = nodes["node_off"]
    for t, name in enumerate(TREES):
        sl = slice(noff[t], noff[t + 1])
        for f in TREE[:-1] + MOM:
            assert np.array_equal(nodes[f][sl], bh_arrays[f"tree_{name}_{f}"]), (name, f)
        assert np.array_equal(nodes["prim_order"][off[t]:off[t + 1]], bh_arrays[f"tree_{name}_prim_order"])


def test_far_field_bitwise(gpu, bh_arrays):
    trees = {}
    for dist, na, nb, quad, want in bh_arrays["ff_values"]:
        key = int(dist)
        if key not in trees:
            trees[key] = (lc.build_moment_tree(bh_arrays[f"ff_{key}_a"]), lc.build_moment_tree(bh_arrays[f"ff_{key}_b"]))
        a, b = trees[key]
        got = lc.far_field_eval(MomentNode(a, int(na)), MomentNode(b, int(nb)), "quadrupole" if quad else "dipole")
        assert got == want, (dist, na, nb, quad)


def test_barnes_hut_matches_reference(gpu, bh_golden, bh_arrays):
    for g in bh_golden["bh"]:
        name = g["name"]
        params = lc.BarnesHutParams(**g["params"])
        a, b = lc.build_moment_tree(bh_arrays[f"bh_{name}_a"]), lc.build_moment_tree(bh_arrays[f"bh_{name}_b"])
        r = lc.barnes_hut_detailed(a, b, params)
        assert abs(r.value - g["value"]) <= 1e-12 * max(1.0, abs(g["value"])), name
        assert r.e_estimate == pytest.approx(g["e_estimate"], rel=1e-13, abs=1e-300), name
        assert r.reran == g["reran"], name
        assert r.beta_used == pytest.approx(g["beta_used"], rel=1e-13), name
        assert lc.link_barnes_hut(a, b, params) == pytest.approx(r.value, abs=1e-15)


def test_visits_match_oracle_traversal(gpu, bh_oracle, bh_arrays):
    """Same set of far-field and leaf decisions as the reference's depth-first walk."""
    for name in ("hopf32", "wobbly_hopf", "self_pair"):
        va, vb = bh_arrays[f"bh_{name}_a"], bh_arrays[f"bh_{name}_b"]
        oa, ob = bh_oracle.Tree(va), bh_oracle.Tree(vb)
        for beta in (1.0, 2.0, 5.0):
            lam_o, est_o, n_far, n_leaf = bh_oracle.dual_eval(oa, ob, beta)
            fa = gpu.bh_forest(va, [0, len(va)])
            fb = gpu.bh_forest(vb, [0, len(vb)])
            lam, est, visits = fa.eval(fb, [[0, 0]], beta)
            # every visited node pair is far, leaf or split; splits = (visits - 1) / 2 for a binary walk
            n_split = (visits - 1) // 2
            assert visits == n_far + n_leaf + n_split, (name, beta)
            assert abs(lam[0] - lam_o) <= 1e-12 and est[0] == pytest.approx(est_o, rel=1e-13)


def test_batched_pairs_equal_single_pairs(gpu, bh_arrays):
    loops = [bh_arrays[k] for k in ("bh_hopf32_a", "bh_hopf32_b", "bh_wobbly_hopf_a", "bh_wobbly_hopf_b",
                                    "bh_arcs_far_a", "bh_arcs_far_b")]
    pairs = [(0, 1), (0, 2), (1, 3), (2, 3), (2, 2), (4, 5), (0, 5)]
    for params in (lc.BarnesHutParams(), lc.BarnesHutParams(e_target=1e-3), lc.BarnesHutParams(order="dipole")):
        value, est, beta, reran = barneshut.evaluate_pairs(loops, pairs, params)
        trees = [lc.build_moment_tree(lp) for lp in loops]
        for k, (i, j) in enumerate(pairs):
            r = lc.barnes_hut_detailed(trees[i], trees[j], params)
            assert abs(value[k] - r.value) <= 1e-12, (i, j)
            assert est[k] == pytest.approx(r.e_estimate, rel=1e-13)
            assert beta[k] == pytest.approx(r.beta_used, rel=1e-13) and reran[k] == r.reran


def test_compute_link_bh(gpu):
    a = _circle(32)
    b = _circle(32, center=(1.0, 0.0, 0.0), u=(0.0, 0.0, 1.0), v=(1.0, 0.0, 0.0))
    diag = {}
    assert lc.compute_link(a, b, lc.KernelChoice(method="bh"), diag) == 1
    assert set(diag) == {"e_estimate", "beta_used", "reran", "raw"}
    with pytest.raises(NotImplementedError):
        lc.compute_link(a, b, lc.KernelChoice(method="cc"))


@pytest.mark.parametrize("name", ["grid4", "e4in1_6x6", "kusari_small", "e4in1_6x6_tight"])
def test_certificate_with_bh_matches_reference(gpu, bh_golden, bh_arrays, name):
    import cases

    g = bh_golden["matrices"][name]
    model = {"grid4": lambda: lc.generators.square_link_grid(4)[0],
             "e4in1_6x6": lambda: lc.generators.european_4in1(6, 6),
             "kusari_small": lambda: lc.generators.kusari_tube(n_around=12, rows=4, partial=5)}[g["model"]]()
    assert cases.fingerprint(model) == g["fingerprint"]
    choice = lc.KernelChoice(method="bh", bh=lc.BarnesHutParams(**g["bh_params"]))
    mat = lc.compute_linking_matrix(model, choice=choice)
    assert np.array_equal(np.array(mat.entries, dtype=np.int64).reshape(-1, 3), bh_arrays[f"mat_{name}_entries"])
    assert mat.kernel_tag == g["kernel_tag"] and mat.model_digest == g["digest"]
    want = g["diagnostics"]
    got = {f"{i},{j}": d for (i, j), d in mat.diagnostics.items()}
    assert set(got) == set(want)
    for k, d in want.items():
        assert list(got[k]) == ["e_estimate", "beta_used", "reran", "raw"]
        assert got[k]["reran"] and got[k]["beta_used"] == pytest.approx(d["beta_used"], rel=1e-13)
        assert got[k]["raw"] == pytest.approx(d["raw"], abs=1e-12)
    # verify with the same kernel: the certificate passes on its own model
    assert lc.verify(model, mat, choice=choice).status == "Pass"


# ---- test_barneshut.py behaviour (reference tests, run on the GPU path) ----

def _leaves(node):
    if node.is_leaf:
        return [node]
    a, b = node.children()
    return _leaves(a) + _leaves(b)


def test_leaf_moments(gpu):
    tree = lc.build_moment_tree(_circle(16, radius=2.0))
    for leaf in _leaves(tree.root):
        a, b = leaf.segment()
        d = b - a
        assert np.allclose(leaf.c_m, d)
        assert np.allclose(leaf.c_d, 0.0, atol=1e-12)
        assert np.allclose(leaf.c_q, np.einsum("i,j,k->ijk", d, d, d) / 12.0, atol=1e-12)


def test_internal_moments_match_direct_sums(gpu):
    rng = np.random.default_rng(2)
    pts = _circle(64, radius=3.0) + 0.2 * rng.normal(size=(64, 3))
    tree = lc.build_moment_tree(pts)
    root = tree.root
    d = tree.seg_b - tree.seg_a
    rho = 0.5 * (tree.seg_a + tree.seg_b) - root.center
    assert np.allclose(root.c_m, d.sum(axis=0), atol=1e-10)
    assert np.allclose(root.c_d, np.einsum("si,sj->ij", d, rho), atol=1e-10)
    cq = np.einsum("si,sj,sk->ijk", d, rho, rho) + np.einsum("si,sj,sk->ijk", d, d, d) / 12.0
    assert np.allclose(root.c_q, cq, atol=1e-10)


def test_root_monopole_vanishes_for_closed_loops(gpu):
    for pts in (_circle(50), _circle(33, radius=7.0, center=(4.0, 1.0, -2.0))):
        tree = lc.build_moment_tree(pts)
        assert np.linalg.norm(tree.root.c_m) < 1e-12 * tree.loop_length


def test_huge_beta_equals_direct_summation(gpu):
    model, _ = lc.generators.torus_link(2, 3, n=256)
    a, b = model.loops[0].start_points(), model.loops[1].start_points()
    params = lc.BarnesHutParams(beta_init=1e6, beta_max=1e6, adaptive=False)
    got = lc.link_barnes_hut(lc.build_moment_tree(a), lc.build_moment_tree(b), params)
    assert got == pytest.approx(lc.link_direct(a, b), abs=1e-12)


def test_accuracy_improves_with_beta(gpu):
    model, _ = lc.generators.double_helix_ribbon(5, 1200)
    trees = [lc.build_moment_tree(lp.start_points()) for lp in model.loops]
    errs = [abs(lc.barnes_hut_detailed(*trees, lc.BarnesHutParams(beta_init=b, beta_max=b, adaptive=False)).value - 5.0)
            for b in (2.0, 8.0, 32.0)]
    assert errs[0] > errs[1] > errs[2]


def test_adaptive_rerun_reduces_error(gpu):
    model, _ = lc.generators.double_helix_ribbon(8, 1500)
    trees = [lc.build_moment_tree(lp.start_points()) for lp in model.loops]
    fixed = lc.barnes_hut_detailed(*trees, lc.BarnesHutParams(beta_init=1.0, beta_max=1.0, adaptive=False))
    adaptive = lc.barnes_hut_detailed(*trees, lc.BarnesHutParams(beta_init=1.0, beta_max=10.0, e_target=1e-3))
    assert adaptive.reran and adaptive.beta_used > 1.0
    assert abs(adaptive.value - 8.0) < abs(fixed.value - 8.0)
    assert fixed.e_estimate > 0.0


def test_large_ribbon_bh_vs_direct(gpu):
    """A 100k x 100k ribbon: Barnes-Hut within its error estimate of the exact link, far fewer node pairs."""
    model, _ = lc.generators.double_helix_ribbon(10, 100_000)
    a, b = (lp.start_points() for lp in model.loops)
    r = lc.barnes_hut_detailed(lc.build_moment_tree(a), lc.build_moment_tree(b))
    assert round(r.value) == 10 and abs(r.value - 10.0) < 0.05


def test_empty_loop_rejected(gpu):
    with pytest.raises(ValueError):
        lc.build_moment_tree(np.zeros((0, 3)))
    with pytest.raises(_native.NativeError):
        gpu.bh_forest(np.zeros((4, 3)), [0, 2, 2, 4])


def _random_loops(seed):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(12):
        n = int(rng.integers(3, 300))
        kind = k % 4
        if kind == 0:      # random walk
            v = np.cumsum(rng.normal(size=(n, 3)), axis=0)
        elif kind == 1:    # integer lattice walk: many equal centers (tie breaking)
            v = np.cumsum(rng.integers(-1, 2, size=(n, 3)), axis=0).astype(float)
        elif kind == 2:    # repeated vertices (zero-length segments) and a flat loop
            v = np.repeat(rng.normal(size=(n // 2 + 2, 3)), 2, axis=0)
            v[:, 2] = 0.0
        else:              # noisy circle with signed zeros
            v = _circle(n, radius=float(rng.uniform(0.5, 5))) + 1e-3 * rng.normal(size=(n, 3))
            v[::7, 1] = -0.0
        out.append(np.ascontiguousarray(v))
    return out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_trees_bitwise_vs_oracle(gpu, bh_oracle, seed):
    loops = _random_loops(seed)
    off = np.zeros(len(loops) + 1, dtype=np.int64)
    np.cumsum([len(v) for v in loops], out=off[1:])
    nodes = gpu.bh_forest(np.concatenate(loops), off).nodes()
    noff = nodes["node_off"]
    for t, v in enumerate(loops):
        o = bh_oracle.Tree(v)
        sl = slice(noff[t], noff[t + 1])
        for f in ("node_lo", "node_hi", "left", "right", "start", "end") + MOM:
            assert np.array_equal(nodes[f][sl], getattr(o, f)), (seed, t, f)
        assert np.array_equal(nodes["prim_order"][off[t]:off[t + 1]], o.prim_order)


@pytest.mark.parametrize("seed", [0, 1])
def test_random_pairs_bh_vs_oracle(gpu, bh_oracle, seed):
    loops = _random_loops(seed)[:6]
    trees = [bh_oracle.Tree(v) for v in loops]
    pairs = [(i, j) for i in range(len(loops)) for j in range(len(loops)) if (i + j) % 2 == 0]
    for beta, quad in ((1.0, True), (2.0, False), (3.5, True)):
        off = np.zeros(len(loops) + 1, dtype=np.int64)
        np.cumsum([len(v) for v in loops], out=off[1:])
        f = gpu.bh_forest(np.concatenate(loops), off)
        lam, est, _ = f.eval(f, pairs, beta, quad)
        for k, (i, j) in enumerate(pairs):
            lo, eo, _, _ = bh_oracle.dual_eval(trees[i], trees[j], beta, quad)
            assert abs(lam[k] - lo) <= 1e-12 * max(1.0, abs(lo)), (seed, i, j, beta)
            assert est[k] == pytest.approx(eo, rel=1e-12, abs=1e-300)
