"""The fused path's pass-1 check (does any segment box of a candidate pair overlap,
discretize.py:151-159 "anything marked") through the 8-segment group boxes.

Pairs of linked rings with segment counts on both sides of the group size (3 … 256,
partial last groups included), the wires at distances from touching to clear and
at random phases: the fused path must be taken exactly when the reference's pass 1
marks nothing (the oracle's segment-box overlap test on the same boxes) and every
pair is within the brute-force limit, and the certificate must equal the oracle's
either way (refinement and large pairs run on the staged path).
"""

import numpy as np
import pytest

import paper_2106_12655_b200 as lc
from paper_2106_12655_b200.certify import run_device_pipeline

pytestmark = pytest.mark.gpu

SIZES = [(3, 5), (7, 9), (8, 8), (9, 17), (15, 16), (31, 33), (63, 65), (64, 64), (100, 7), (255, 256),
         (256, 256)]
FACTORS = [0.02, 0.1, 0.4, 1.5, 6.0]   # radius of the second ring / segment length of the first


def _radii(na):
    return [min(0.9, f * 2.0 * np.pi / na) for f in FACTORS]


def _ring(n, center, u, v, radius, phase):
    th = phase + 2.0 * np.pi * np.arange(n) / n
    return np.asarray(center) + radius * (np.outer(np.cos(th), u) + np.outer(np.sin(th), v))


def _pair_model(na, nb, rb, rng):
    ex, ey, ez = np.eye(3)
    a = _ring(na, (0.0, 0.0, 0.0), ex, ey, 1.0, rng.uniform(0, 2 * np.pi))
    b = _ring(nb, (1.0, 0.0, 0.2 * rb), ex, ez, rb, rng.uniform(0, 2 * np.pi))
    return lc.CurveModel([lc.LoopGeometry.from_polyline(a), lc.LoopGeometry.from_polyline(b)])


def _pierced_model(na, nb, k, rng):
    """A small ring around segment k of the first ring (k in the first, a middle
    or the last, possibly partial, 8-segment group): that segment passes through
    its disk, so the two segment boxes there meet for most phases."""
    ex, ey, ez = np.eye(3)
    a = _ring(na, (0.0, 0.0, 0.0), ex, ey, 1.0, rng.uniform(0, 2 * np.pi))
    p, q = a[k], a[(k + 1) % na]
    mid, seg = 0.5 * (p + q), float(np.linalg.norm(q - p))
    radial = mid / np.linalg.norm(mid)
    b = _ring(nb, mid, radial, ez, 0.1 * seg, rng.uniform(0, 2 * np.pi))
    return lc.CurveModel([lc.LoopGeometry.from_polyline(a), lc.LoopGeometry.from_polyline(b)])


def _cases(rng):
    for na, nb in SIZES:
        for rb in _radii(na):
            yield (na, nb, "ring", rb), _pair_model(na, nb, rb, rng)
        for k in sorted({0, 7 % na, 8 % na, na // 2, na - 1}):
            yield (na, nb, "pierced", k), _pierced_model(na, nb, k, rng)


def _oracle_pass1_marks(oracle, model):
    coeffs, t, off = model.packed()
    pairs = oracle.pls(coeffs, t, off)
    lo, hi = oracle.tight_boxes(coeffs, t[:, 0], t[:, 1])
    for i, j in np.asarray(pairs).reshape(-1, 2):
        a, b = slice(off[i], off[i + 1]), slice(off[j], off[j + 1])
        if len(oracle.overlap_pairs(lo[a], hi[a], lo[b], hi[b])):
            return True
    return False


def test_pass1_groups_decide_like_the_reference(oracle, monkeypatch):
    monkeypatch.setenv("LINKCERT_FUSED", "1")
    rng = np.random.default_rng(2106)
    outcomes = {True: 0, False: 0}
    fused = 0
    for case, m in _cases(rng):
        marks = _oracle_pass1_marks(oracle, m)
        outcomes[marks] += 1
        coeffs, t, off = m.packed()
        try:
            want, pairs, raw = oracle.link_matrix(coeffs, t, off, m.xi)
        except oracle.OracleDiscretizationError as e:
            with pytest.raises(lc.DiscretizationError) as got:
                lc.compute_linking_matrix(m)
            assert got.value.kind == e.kind, case
            continue
        used = None
        for _ in range(2):   # a first run past the item capacity sizes it and reruns staged
            p2, r2, _, _, ctx = run_device_pipeline(m)
            used = ctx.last_run_fused()
        # pairs past the reference's brute-force limit (n_i * n_j > 16384, bvh.py:224) are
        # swept on the staged path, checked or not
        small = all(case[0] * case[1] <= 16384 for _ in np.asarray(pairs).reshape(-1, 2))
        assert bool(used) == (small and not marks), (case, marks, used)
        fused += bool(used)
        assert np.array_equal(lc.compute_linking_matrix(m).array, want), case
        assert np.array_equal(np.asarray(p2).reshape(-1, 2), np.asarray(pairs).reshape(-1, 2)), case
        if len(raw):
            assert np.max(np.abs(np.asarray(r2) - raw)) < 1e-9, case
    # both decisions are exercised
    assert outcomes[True] >= 20 and outcomes[False] >= 20, outcomes
    assert fused >= 20, fused
