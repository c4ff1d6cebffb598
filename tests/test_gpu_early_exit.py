"""verify(..., early_exit=True) with the device early exit.

The reference (certify.py:195-216) evaluates the pairs in its ordering —
certificate pairs, then the other candidates, each in key order — and stops at
the first pair whose value differs.  On the fused single-GPU path the library
evaluates in that order and cancels every pair past the first failure found;
the report is replayed from the evaluated pairs.  Checks: the reports equal
the reference's goldens and the staged path's (every pair computed, host
replay), and fewer pairs are evaluated than the candidates.
"""

import warnings

import numpy as np
import pytest

import cases
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native, generators as gen
from paper_2106_12655_b200.geometry import CurveModel, LoopGeometry

pytestmark = pytest.mark.gpu


def _verify(model, cert, **kw):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return lc.verify(model, cert, **kw)


def _same(a, b):
    return (a.status, a.destroyed, a.created, a.changed, a.first_failure) == \
           (b.status, b.destroyed, b.created, b.changed, b.first_failure)


@pytest.mark.parametrize("name", list(cases.edit_cases(full=True)))
def test_device_early_exit_matches_reference(golden, monkeypatch, name):
    g = golden["verify"][name]["early_exit"]
    before, after = cases.edit_cases(full=name.startswith("kusari_full"))[name]
    cert = lc.compute_linking_matrix(before)
    ctx = _native.context()
    rep = _verify(after, cert, early_exit=True)
    assert ctx.last_run_fused() in (1, 2)
    assert rep.status == g["status"] and [list(p) for p in rep.destroyed] == g["destroyed"]
    assert [list(p) for p in rep.created] == g["created"] and [list(p) for p in rep.changed] == g["changed"]
    assert list(rep.first_failure) == g["first_failure"]
    place, n_eval = ctx.early_exit_stats()
    P = len(lc.potential_link_search(after))
    keys = [tuple(e[:2]) for e in cert.entries]
    assert place == keys.index(tuple(g["first_failure"]))          # a certificate pair: its index
    assert 0 <= n_eval < P                                           # pairs past it were cancelled
    monkeypatch.setenv("LINKCERT_FUSED", "0")                        # staged: all pairs, host replay
    assert _same(_verify(after, cert, early_exit=True), rep)


def _ring(c, u, v, n=48, r=1.0):
    t = np.linspace(0.0, 2.0 * np.pi, n, endpoint=False)
    return np.asarray(c) + r * np.outer(np.cos(t), u) + r * np.outer(np.sin(t), v)


def test_device_early_exit_on_a_computed_pair(monkeypatch):
    """The first failure is a pair that is still a candidate (a reversed ring flips
    its links): it is found by the Gauss kernel, not before it."""
    ks = gen.kusari_tube(n_around=12, rows=4, partial=5)
    pts = [lp.control_points.copy() for lp in ks.loops]
    n_big = 12 * 4 + 5
    pts[n_big + 30] = pts[n_big + 30][::-1].copy()
    after = CurveModel([LoopGeometry.from_polyline(p) for p in pts])
    cert = lc.compute_linking_matrix(ks)
    rep = _verify(after, cert, early_exit=True)
    assert rep.status == "Aborted" and len(rep.changed) == 1 and rep.first_failure == rep.changed[0]
    place, n_eval = _native.context().early_exit_stats()
    assert place == [tuple(e[:2]) for e in cert.entries].index(rep.first_failure)
    full = _verify(after, cert)
    assert rep.first_failure == min(full.changed)                    # first in the certificate's order
    monkeypatch.setenv("LINKCERT_FUSED", "0")
    assert _same(_verify(after, cert, early_exit=True), rep)


def test_device_early_exit_created_link_and_pass(monkeypatch):
    """A new link (not in the certificate) is ordered after every certificate pair;
    an unchanged model evaluates every pair and passes."""
    ex, ey, ez = np.eye(3)
    loops = [_ring((4.0 * k, 0, 0), ex, ey) for k in range(6)] + [_ring((4.0 * k + 1.0, 0, 0), ez, ex)
                                                                for k in range(0, 6, 2)]
    loops.append(_ring((40.0, 0, 0), ez, ex))                        # far: links nothing
    before = CurveModel([LoopGeometry.from_polyline(p) for p in loops])
    cert = lc.compute_linking_matrix(before)
    assert len(cert.entries) == 3
    moved = list(loops)
    moved[-1] = _ring((4.0 * 5 + 1.0, 0, 0), ez, ex)                # now links ring 5
    after = CurveModel([LoopGeometry.from_polyline(p) for p in moved])
    rep = _verify(after, cert, early_exit=True)
    assert rep.status == "Aborted" and rep.created == [(5, 9)] and rep.first_failure == (5, 9)
    place, n_eval = _native.context().early_exit_stats()
    assert place >= len(cert.entries)                                # after the certificate's pairs
    monkeypatch.setenv("LINKCERT_FUSED", "0")
    assert _same(_verify(after, cert, early_exit=True), rep)
    monkeypatch.delenv("LINKCERT_FUSED")
    ok = _verify(before, cert, early_exit=True)
    assert ok.status == "Pass"
    place, n_eval = _native.context().early_exit_stats()
    assert place == -1 and n_eval == len(lc.potential_link_search(before))
