"""Pin the CPU oracle against vectors produced by the reference itself (tests/golden/).

CPU only.  The C Gauss-sum oracle runs the reference's IEEE operation
sequence (no FMA, fastmath=False numba), so raw values must be BITWISE equal;
PLS pairs, discretized vertices, certificates and verify lists are exact.
"""

import hashlib

import numpy as np
import pytest

import cases


def test_pair_lambda_bitwise(oracle, golden_arrays):
    q = golden_arrays["quads"]
    want = golden_arrays["quads_lambda"]
    got = np.array([oracle.pair_lambda(r[0:3], r[3:6], r[6:9], r[9:12]) for r in q])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name", list(cases.link_cases()))
def test_link_direct_bitwise(oracle, golden, name):
    g = golden["links"][name]
    m = cases.link_cases()[name]
    assert cases.fingerprint(m) == g["fingerprint"]
    a, b = (lp.start_points() for lp in m.loops)
    assert oracle.link_direct(a, b, "atan") == g["atan"]
    assert oracle.link_direct(a, b, "anglesum") == g["anglesum"]
    assert oracle.link_direct(b, a, "atan") == g["atan_swapped"]


@pytest.mark.parametrize("k", range(4))
def test_link_direct_random_polygons_bitwise(oracle, golden, golden_arrays, k):
    a, b = golden_arrays[f"rand_a{k}"], golden_arrays[f"rand_b{k}"]
    assert oracle.link_direct(a, b, "atan") == golden["links"][f"random_{k}"]["atan"]
    assert oracle.link_direct(a, b, "anglesum") == golden["links"][f"random_{k}"]["anglesum"]


SMALL = [n for n in cases.cert_models() if n != "kusari_full"]


@pytest.mark.parametrize("name", SMALL + ["kusari_full"])
def test_pls_discretize_certificate(oracle, golden, golden_arrays, name):
    g = golden["certs"][name]
    m = cases.cert_models(full=name == "kusari_full")[name]
    assert cases.fingerprint(m) == g["fingerprint"]
    assert m.xi == g["xi"]
    coeffs, t, off = m.packed()
    pairs = oracle.pls(coeffs, t, off)
    assert np.array_equal(pairs, golden_arrays[f"{name}__pairs"])
    verts, voff = oracle.discretize(coeffs, t, off, m.xi, pairs)
    assert len(verts) == g["discretized_vertices"]
    assert hashlib.sha256(verts.tobytes()).hexdigest() == g["discretized_sha256"]
    raw = oracle.evaluate_pairs(verts, voff, pairs)
    lk = np.array([oracle.round_link(r)[0] for r in raw], dtype=np.int64)
    keep = lk != 0
    entries = np.concatenate([pairs[keep], lk[keep, None]], axis=1)
    assert np.array_equal(entries, golden_arrays[f"{name}__entries"])


@pytest.mark.parametrize("name", list(cases.disc_error_cases()))
def test_discretize_errors(oracle, golden, golden_arrays, name):
    g = golden["discretize"][name]
    m, prs, kw = cases.disc_error_cases()[name]
    assert cases.fingerprint(m) == g["fingerprint"]
    coeffs, t, off = m.packed()
    if g["ok"]:
        verts, _ = oracle.discretize(coeffs, t, off, m.xi, prs, **kw)
        assert np.array_equal(verts, golden_arrays[f"disc_{name}__verts"])
    else:
        with pytest.raises(oracle.OracleDiscretizationError) as e:
            oracle.discretize(coeffs, t, off, m.xi, prs, **kw)
        assert e.value.kind == g["kind"]
        assert list(e.value.loops) == g["loops"]
        assert str(e.value) == g["message"]


@pytest.mark.parametrize("name", ["grid6_pull", "e4in1_32x32_pull165", "kusari_small_after"])
def test_verify_lists(oracle, golden, golden_arrays, name):
    g = golden["verify"][name]
    before, after = cases.edit_cases()[name]
    assert cases.fingerprint(after) == g["after_fingerprint"]
    coeffs, t, off = after.packed()
    entries, _, _ = oracle.link_matrix(coeffs, t, off, after.xi)
    assert np.array_equal(entries, golden_arrays[f"{name}__after_entries"])
    bc, bt, bo = before.packed()
    before_entries, _, _ = oracle.link_matrix(bc, bt, bo, before.xi)
    ref = {(int(i), int(j)): int(v) for i, j, v in before_entries}
    got = {(int(i), int(j)): int(v) for i, j, v in entries}
    destroyed, created, changed = oracle.diff(ref, got)
    assert [list(p) for p in destroyed] == g["full"]["destroyed"]
    assert [list(p) for p in created] == g["full"]["created"]
    assert [list(p) for p in changed] == g["full"]["changed"]


@pytest.mark.parametrize("name", list(cases.validation_cases()))
def test_chord_validation_errors(oracle, golden, name):
    """Chords that fail PolylineLoop validation without refinement (golden from the reference)."""
    g = golden["validation"][name]
    m = cases.validation_cases()[name]
    assert cases.fingerprint(m) == g["fingerprint"]
    coeffs, t, off = m.packed()
    assert [list(p) for p in oracle.pls(coeffs, t, off)] == g["pairs"]
    with pytest.raises(oracle.OracleValidationError) as e:
        oracle.discretize(coeffs, t, off, m.xi, [tuple(p) for p in g["pairs"]])
    assert not g["ok"] and str(e.value) == g["message"]
