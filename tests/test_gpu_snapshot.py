"""The model snapshot paths on the GPU: loops built one by one (per-loop vertex
pointers, gathered by the library), the bulk block, a mixed model (a generic
loop forces the packed-coefficient upload) and a reassigned loop all give the
bitwise same certificate / raw sums as the oracle-pinned bulk path."""

import warnings

import numpy as np
import pytest

import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import generators as gen, model_io, workloads
from paper_2106_12655_b200.certify import run_device_pipeline

pytestmark = pytest.mark.gpu


def _results(m):
    return [np.array(a).copy() for a in run_device_pipeline(m)[:4]]


def test_per_loop_upload_equals_bulk():
    v, off = workloads.kusari_tube_vertices(n_around=24, rows=6, partial=9)
    bulk = lc.CurveModel.from_polyline_arrays(v, off)
    loops = [lc.LoopGeometry.from_polyline(v[off[k]:off[k + 1]]) for k in range(len(off) - 1)]
    fresh = lc.CurveModel(loops)
    assert fresh.snapshot().poly and fresh.xi == bulk.xi
    want = _results(bulk)
    for got in (_results(fresh), _results(lc.CurveModel(list(loops), xi=bulk.xi))):
        for a, b in zip(want, got):
            assert np.array_equal(a, b)
    assert model_io.model_digest(fresh) == model_io.model_digest(bulk) == model_io.model_digest_python(fresh)


def test_mixed_and_reassigned_models_take_the_packed_upload():
    m = gen.kusari_tube(n_around=12, rows=4, partial=5)
    want = lc.compute_linking_matrix(m)
    loops = list(m.loops)
    loops[7] = lc.LoopGeometry(loops[7].coeffs, loops[7].t)      # same arrays, generic constructor
    mixed = lc.CurveModel(loops, xi=m.xi)
    assert not mixed.snapshot().poly
    got = lc.compute_linking_matrix(mixed)
    assert got.entries == want.entries and got.model_digest == want.model_digest
    # a reassigned loop: tracked, re-uploaded, the certificate follows the new geometry
    pts = [lp.control_points.copy() for lp in m.loops]
    fresh = [lc.LoopGeometry.from_polyline(p) for p in pts]
    model = lc.CurveModel(fresh, xi=m.xi)
    assert lc.compute_linking_matrix(model).entries == want.entries
    k = 60                                                     # a connector ring of the small tube
    c = fresh[k].coeffs.copy()
    c[:, 0, 2] += 50.0                                         # move the ring far away (a0 only: still closed)
    fresh[k].coeffs = c
    after = lc.compute_linking_matrix(model)
    assert after.entries != want.entries
    assert after.model_digest != want.model_digest
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        rep = lc.verify(model, want)
    assert rep.status == "Fail" and rep.destroyed and any("digest" in str(x.message) for x in w)
