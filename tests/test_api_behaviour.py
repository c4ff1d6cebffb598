"""Behaviour of the drop-in API that the reference's own suite pins (test_direct,
test_kernels, test_certify, test_discretize, test_pls), exercised through the
CUDA path: symmetries, variants, errors and warnings, thread independence,
chord placement.  Written against the reference semantics.
"""

from __future__ import annotations

import warnings

import numpy as np
import pytest

import cases
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200.certify import ABORTED, FAIL, PASS

pytestmark = pytest.mark.gpu

EX, EY, EZ = np.eye(3)


def _hopf(n=64):
    return cases.circ(n, (0, 0, 0), EX, EY), cases.circ(n, (1.0, 0, 0), EZ, EX)


def test_link_direct_symmetries_and_variants():
    a, b = _hopf(96)
    base = lc.link_direct(a, b)
    assert round(base) == 1 and abs(base - 1.0) < 1e-12
    assert abs(lc.link_direct(b, a) - base) < 1e-12                 # swap
    assert abs(lc.link_direct(a[::-1].copy(), b) + base) < 1e-12    # one orientation flipped: sign flips
    assert abs(lc.link_direct(a[::-1].copy(), b[::-1].copy()) - base) < 1e-12
    assert abs(lc.link_direct(a, b, variant="anglesum") - base) < 1e-9
    with pytest.raises(ValueError):
        lc.link_direct(a, b, variant="bogus")
    # PolylineLoop objects are accepted like arrays
    assert abs(lc.link_direct(lc.PolylineLoop(a), lc.PolylineLoop(b)) - base) < 1e-15


def test_unlinked_coplanar_loops_are_zero():
    a = cases.circ(64, (0, 0, 0), EX, EY)
    b = cases.circ(64, (3.0, 0, 0), EX, EY)
    assert abs(lc.link_direct(a, b)) < 1e-12


def test_compute_link_rounding_and_diagnostics():
    a, b = _hopf(64)
    diag = {}
    assert lc.compute_link(a, b, diagnostics=diag) == 1
    assert abs(diag["raw"] - 1.0) < 1e-12
    assert lc.KernelChoice().tag == "ds:atan" and lc.KernelChoice(ds_variant="anglesum").tag == "ds:anglesum"


def test_verify_warns_on_digest_mismatch_and_passes():
    model, _ = lc.generators.square_link_grid(4)
    cert = lc.compute_linking_matrix(model)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        assert lc.verify(model, cert).status == PASS        # same digest: no warning
    moved = lc.CurveModel([lc.LoopGeometry.from_polyline(lp.start_points() + np.array([0.0, 0.0, 1e-3]))
                           for lp in model.loops])
    with pytest.warns(UserWarning, match="model digest differs"):
        rep = lc.verify(moved, cert)
    assert rep.status == PASS                                  # a rigid shift keeps every link


def test_verify_loop_count_mismatch_fails():
    model, _ = lc.generators.square_link_grid(4)
    cert = lc.compute_linking_matrix(model)
    smaller = lc.CurveModel(model.loops[:-1])
    rep = lc.verify(smaller, cert)
    assert rep.status == FAIL
    assert rep.message == f"loop count mismatch: model has {smaller.num_loops}, certificate has {model.num_loops}"


def test_verify_early_exit_aborts():
    before, after = cases.edit_cases()["grid6_pull"]
    cert = lc.compute_linking_matrix(before)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        full = lc.verify(after, cert)
        ee = lc.verify(after, cert, early_exit=True)
    assert full.status == FAIL and ee.status == ABORTED
    assert ee.first_failure == min(full.failing_pairs())


def test_thread_count_does_not_change_results():
    model = lc.generators.european_4in1(8, 8)
    ref = lc.compute_linking_matrix(model)
    for threads in (1, 4, 16):
        assert lc.compute_linking_matrix(model, threads=threads) == ref


def test_excluded_pairs_not_reported():
    model, _ = lc.generators.square_link_grid(4)
    full = lc.compute_linking_matrix(model)
    drop = {full.entries[0][:2], full.entries[-1][:2][::-1]}   # either orientation
    part = lc.compute_linking_matrix(model, excluded=drop)
    assert set(full.entries) - set(part.entries) == {full.entries[0], full.entries[-1]}


def test_chord_vertices_lie_on_the_curves():
    """Every discretized vertex is the curve point eval_cubics(coeffs[seg], t) of
    some segment and parameter (here: segment start points after refinement)."""
    m = cases.disc_error_cases()["tight_ok"][0]
    polys = lc.discretize(m, lc.potential_link_search(m))
    for loop, poly in zip(m.loops, polys):
        assert len(poly) >= loop.coeffs.shape[0]
        c = loop.coeffs
        # distance of every chord vertex to the densely sampled curve
        ts = np.linspace(0.0, 1.0, 4097)
        pts = (c[:, None, 0] + c[:, None, 1] * ts[None, :, None] + c[:, None, 2] * ts[None, :, None] ** 2
               + c[:, None, 3] * ts[None, :, None] ** 3).reshape(-1, 3)
        d = np.min(np.linalg.norm(poly.vertices[:, None, :] - pts[None, :, :], axis=2), axis=1)
        assert d.max() < 1e-3


def test_pls_degenerate_models():
    with pytest.raises(lc.ValidationError):
        lc.potential_link_search(lc.CurveModel([]))
    one = lc.CurveModel([lc.LoopGeometry.from_polyline(cases.circ(8, (0, 0, 0), EX, EY))])
    assert len(lc.potential_link_search(one)) == 0
    a, b = _hopf(32)
    hopf = lc.CurveModel([lc.LoopGeometry.from_polyline(a), lc.LoopGeometry.from_polyline(b)])
    assert list(lc.potential_link_search(hopf)) == [(0, 1)]
    assert list(lc.potential_link_search(hopf, excluded={(1, 0)})) == []


def test_concurrent_callers_share_the_context_safely():
    """Two threads certifying different models on the one device context: the
    session lock keeps upload -> pipeline -> result views of a call together."""
    import threading

    models = [lc.generators.european_4in1(8, 8), lc.generators.square_link_grid(6)[0]]
    want = [lc.compute_linking_matrix(m) for m in models]
    errors = []

    def worker(k):
        try:
            for _ in range(20):
                assert lc.compute_linking_matrix(models[k]) == want[k]
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore")
                    assert lc.verify(models[k], want[k]).status == PASS
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(k,)) for k in (0, 1)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
