"""The "anglesum" direct-summation variant on the GPU (GAUSS_ANGLESUM) against the
reference's own anglesum values (linkcert/direct.py:68-134, goldens from
tests/golden/make_golden.py) and the oracle's C restatement of it.

The kernel runs the reference recurrence per outer segment in the reference's
operation order, so every crossing count and normalized phase is the
reference's; the raw sums differ only by the per-row atan2 ulps and the
summation order of the rows (observed <= 1e-14; the bar is RAW_TOL = 1e-9).
"""

import numpy as np
import pytest

import cases
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native

pytestmark = pytest.mark.gpu

RAW_TOL = 1e-9
TIGHT = 1e-12   # what the kernel actually achieves (same recurrence as the reference)


@pytest.mark.parametrize("name", list(cases.link_cases()))
def test_anglesum_vs_reference_goldens(gpu, golden, name):
    g = golden["links"][name]
    m = cases.link_cases()[name]
    assert cases.fingerprint(m) == g["fingerprint"]
    a, b = (lp.start_points() for lp in m.loops)
    raw = lc.link_direct(a, b, variant="anglesum")
    assert abs(raw - g["anglesum"]) < TIGHT
    assert round(raw) == round(g["anglesum"])
    assert gpu.link_direct(a, b, _native.GAUSS_ANGLESUM) == raw


@pytest.mark.parametrize("k", range(4))
def test_anglesum_random_polygons(gpu, golden, golden_arrays, k):
    """Self-intersecting random polygons: every crossing-count branch of _link_angle_sum."""
    a, b = golden_arrays[f"rand_a{k}"], golden_arrays[f"rand_b{k}"]
    assert abs(lc.link_direct(a, b, variant="anglesum") - golden["links"][f"random_{k}"]["anglesum"]) < TIGHT


def test_anglesum_vs_oracle_seeded(gpu, oracle):
    rng = np.random.default_rng(5)
    worst = 0.0
    for k in range(12):
        n1, n2 = int(rng.integers(3, 300)), int(rng.integers(3, 300))
        a = rng.normal(size=(n1, 3)) * 10.0 ** rng.uniform(-3, 3)
        b = rng.normal(size=(n2, 3)) * 10.0 ** rng.uniform(-3, 3) + rng.normal(size=3)
        got = lc.link_direct(a, b, variant="anglesum")
        want = oracle.link_direct(a, b, "anglesum")
        worst = max(worst, abs(got - want))
    assert worst < TIGHT


def test_anglesum_long_rows(gpu, oracle):
    """One pair with 5,000 inner segments per outer row (the kernel walks each row in order)."""
    m, _ = lc.generators.double_helix_ribbon(3, 5000)
    a, b = (lp.control_points for lp in m.loops)
    got = lc.link_direct(a, b, variant="anglesum")
    assert abs(got - oracle.link_direct(a, b, "anglesum")) < TIGHT
    assert abs(got - 3.0) < RAW_TOL


def test_anglesum_certificate_and_verify(gpu, golden, golden_arrays):
    models = cases.cert_models()
    m = models["kusari_small"]
    choice = lc.KernelChoice(ds_variant="anglesum")
    mat = lc.compute_linking_matrix(m, choice=choice)
    assert mat.kernel_tag == "ds:anglesum"
    assert np.array_equal(mat.array, golden_arrays["kusari_small__entries"])
    ref = lc.compute_linking_matrix(m)
    assert np.array_equal(mat.array, ref.array) and mat.model_digest == ref.model_digest
    rep = lc.verify(m, ref, choice=choice)
    assert rep.status == "Pass"


def test_anglesum_evaluate_and_staged_items(gpu):
    """Sequential (whole-row) items are built per mode; running another mode on them is refused."""
    m, _ = lc.generators.torus_link(2, 3, n=300)
    a, b = (lp.control_points for lp in m.loops)
    verts = np.concatenate([a, b])
    off = np.array([0, len(a), len(a) + len(b)], dtype=np.int64)
    pairs = np.array([[0, 1]], dtype=np.int32)
    n_seq = gpu.stage_polylines(verts, off, pairs, _native.GAUSS_ANGLESUM)
    assert n_seq == (300 + 31) // 32
    with pytest.raises(_native.NativeError):
        gpu.gauss_run(_native.GAUSS_PHASE, 0, n_seq)
    gpu.gauss_run(_native.GAUSS_ANGLESUM, 0, n_seq)
    raw, lk, flags = gpu.gauss_reduce()
    assert lk[0] == 6 and flags[0] == 0
    assert raw[0] == lc.link_direct(a, b, variant="anglesum")
