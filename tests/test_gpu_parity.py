"""Parity of the sm_100a path (through the C-ABI) with the reference goldens and the oracle.

Bars (BASELINE.json north_star): integer linking numbers, PLS pair sets,
discretized vertices and verify lists bit-exact; raw per-pair sums within
RAW_TOL = 1e-9 absolute.
"""

import hashlib
import warnings

import numpy as np
import pytest

import cases
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native
from paper_2106_12655_b200.certify import ABORTED, FAIL, PASS

pytestmark = pytest.mark.gpu

RAW_TOL = 1e-9
MODES = [_native.GAUSS_PHASE, _native.GAUSS_ATAN, _native.GAUSS_REF]


def test_segment_pair_lambda(gpu, golden_arrays):
    q = golden_arrays["quads"]
    got = gpu.segment_pair_lambda(q)
    want = golden_arrays["quads_lambda"]
    assert np.max(np.abs(got - want)) < 1e-13
    assert lc.segment_pair_lambda(q[0, 0:3], q[0, 3:6], q[0, 6:9], q[0, 9:12]) == pytest.approx(want[0], abs=1e-15)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", list(cases.link_cases()))
def test_link_direct_modes(gpu, golden, name, mode):
    g = golden["links"][name]
    m = cases.link_cases()[name]
    assert cases.fingerprint(m) == g["fingerprint"]
    a, b = (lp.start_points() for lp in m.loops)
    raw = gpu.link_direct(a, b, mode)
    assert abs(raw - g["atan"]) < RAW_TOL
    assert round(raw) == round(g["atan"])
    assert abs(gpu.link_direct(b, a, mode) - g["atan_swapped"]) < RAW_TOL


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("k", range(4))
def test_random_polygons(gpu, golden, golden_arrays, k, mode):
    a, b = golden_arrays[f"rand_a{k}"], golden_arrays[f"rand_b{k}"]
    assert abs(gpu.link_direct(a, b, mode) - golden["links"][f"random_{k}"]["atan"]) < RAW_TOL


ALL_CERTS = list(cases.cert_models(full=True))


@pytest.fixture(scope="module")
def cert_models():
    return cases.cert_models(full=True)


@pytest.mark.parametrize("name", ALL_CERTS)
def test_pls_pairs_exact(golden, golden_arrays, cert_models, name):
    m = cert_models[name]
    assert cases.fingerprint(m) == golden["certs"][name]["fingerprint"]
    pl = lc.potential_link_search(m)
    assert np.array_equal(pl.array, golden_arrays[f"{name}__pairs"])


@pytest.mark.parametrize("n_loops,spread", [(300, 3.0), (2000, 40.0), (40000, 400.0)])
def test_pls_dense_and_large_vs_oracle(oracle, n_loops, spread):
    """Crowded boxes (> 16 later overlaps per loop: two-pass fallback) and L > 32768 (sweep path)."""
    rng = np.random.default_rng(n_loops)
    ex, ey, ez = np.eye(3)
    centers = rng.uniform(0, spread, size=(n_loops, 3))
    pts = np.stack([cases.circ(6, c, ex, ey if k % 2 else ez, 0.5 + 0.5 * rng.random())
                    for k, c in enumerate(centers)])
    off = np.arange(n_loops + 1, dtype=np.int64) * 6
    m = lc.CurveModel.from_polyline_arrays(pts.reshape(-1, 3), off)
    coeffs, t, o = m.packed()
    want = oracle.pls(coeffs, t, o) if n_loops <= 2000 else None
    got = lc.potential_link_search(m).array
    if want is not None:
        assert np.array_equal(got, want)
    else:   # large L: check soundness/completeness on a random sample of rows against brute force
        lo, hi = oracle.loop_boxes(coeffs, t, o)
        for i in rng.choice(n_loops, 50, replace=False):
            ov = np.all((lo[i] <= hi) & (lo <= hi[i]), axis=1)
            ov[: i + 1] = False
            assert np.array_equal(np.nonzero(ov)[0], got[got[:, 0] == i, 1])


def test_pls_sweep_path_exact(golden_arrays):
    """The sort-and-sweep PLS (used for L > 32768) gives the same pair sets."""
    import subprocess
    import sys

    code = (
        "import sys, numpy as np; sys.path.insert(0, 'tests'); import cases, paper_2106_12655_b200 as lc\n"
        "g = np.load('tests/golden/golden_arrays.npz')\n"
        "for name, m in cases.cert_models(full=True).items():\n"
        "    assert np.array_equal(lc.potential_link_search(m).array, g[name + '__pairs']), name\n"
        "print('sweep ok')\n")
    env = dict(__import__("os").environ, LINKCERT_PLS_SWEEP="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "sweep ok" in out.stdout, out.stderr[-2000:]


@pytest.mark.parametrize("name", ALL_CERTS)
def test_discretize_bitwise(golden, golden_arrays, cert_models, name):
    m = cert_models[name]
    polys = lc.discretize(m, lc.potential_link_search(m))
    verts = np.concatenate([p.vertices for p in polys])
    assert len(verts) == golden["certs"][name]["discretized_vertices"]
    assert hashlib.sha256(verts.tobytes()).hexdigest() == golden["certs"][name]["discretized_sha256"]


@pytest.mark.parametrize("name", ALL_CERTS)
def test_certificate_exact(golden, golden_arrays, cert_models, name):
    m = cert_models[name]
    timings = {}
    mat = lc.compute_linking_matrix(m, timings=timings)
    assert np.array_equal(mat.array, golden_arrays[f"{name}__entries"])
    assert mat.model_digest == golden["certs"][name]["digest"]
    assert mat.kernel_tag == "ds:atan"
    assert {"pls", "discretize", "kernel"} <= set(timings)


@pytest.mark.parametrize("name", ["grid6_pull", "e4in1_32x32_pull165", "kusari_small_after", "kusari_full_after"])
def test_verify_reports_exact(golden, name):
    g = golden["verify"][name]
    before, after = cases.edit_cases(full=name.startswith("kusari_full"))[name]
    assert cases.fingerprint(after) == g["after_fingerprint"]
    cert = lc.compute_linking_matrix(before)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        rep = lc.verify(after, cert)
        rep_ee = lc.verify(after, cert, early_exit=True)
    for r, want in ((rep, g["full"]), (rep_ee, g["early_exit"])):
        assert r.status == want["status"]
        assert [list(p) for p in r.destroyed] == want["destroyed"]
        assert [list(p) for p in r.created] == want["created"]
        assert [list(p) for p in r.changed] == want["changed"]
        assert (list(r.first_failure) if r.first_failure else None) == want["first_failure"]
    assert lc.verify(before, cert).status == PASS


@pytest.mark.parametrize("name", list(cases.disc_error_cases()))
def test_discretize_errors(golden, golden_arrays, name):
    g = golden["discretize"][name]
    m, prs, kw = cases.disc_error_cases()[name]
    params = lc.DiscretizationParams(**kw)
    if g["ok"]:
        polys = lc.discretize(m, lc.PairList(tuple(prs)), params)
        assert np.array_equal(np.concatenate([p.vertices for p in polys]), golden_arrays[f"disc_{name}__verts"])
    else:
        with pytest.raises(lc.DiscretizationError) as e:
            lc.discretize(m, lc.PairList(tuple(prs)), params)
        assert e.value.kind == g["kind"]
        assert list(e.value.loops) == g["loops"]
        assert str(e.value) == g["message"]


def test_raw_parity_vs_oracle_seeded(gpu, oracle):
    """Seeded random loop batches: raw within RAW_TOL, integers exact, every mode."""
    rng = np.random.default_rng(7)
    loops = [rng.normal(size=(int(n), 3)) * 2.0 for n in rng.integers(3, 300, size=40)]
    off = np.concatenate([[0], np.cumsum([len(x) for x in loops])]).astype(np.int64)
    verts = np.concatenate(loops)
    pairs = np.array([(i, j) for i in range(40) for j in range(i + 1, 40)], dtype=np.int32)
    want = oracle.evaluate_pairs(verts, off, pairs)
    for mode in MODES:
        raw, lk, flags = gpu.evaluate_pairs(verts, off, pairs, mode)
        assert np.max(np.abs(raw - want)) < RAW_TOL
        ok = np.abs(want - np.round(want)) <= 0.25
        assert np.array_equal(lk[ok], np.round(want[ok]).astype(np.int64))


def test_deterministic_and_split_invariant(gpu):
    """Bitwise identical raw sums run to run and for any split of the item range (multi-GPU contract)."""
    import torch

    m = lc.generators.kusari_tube(n_around=24, rows=8, partial=10)
    coeffs, t, off = m.packed()
    gpu.upload_model(coeffs, t, off)
    gpu.run_pipeline(None, m.xi, 2.220446049250313e-16, 64, 1 << 22)
    raw0, lk0, _ = gpu.get_results()
    raw1, lk1, _ = gpu.evaluate_staged(_native.GAUSS_PHASE)
    assert np.array_equal(raw0.view(np.int64), raw1.view(np.int64))
    n = gpu.prepare_gauss()
    for world in (2, 3, 8):
        buf = torch.zeros(n, dtype=torch.float64, device="cuda")
        bounds = gpu.shard_bounds(world)
        for r in range(world):
            gpu.gauss_run(_native.GAUSS_PHASE, int(bounds[r]), int(bounds[r + 1]), buf.data_ptr())
        gpu.synchronize()
        raw2, lk2, _ = gpu.gauss_reduce(buf.data_ptr())
        assert np.array_equal(raw0.view(np.int64), raw2.view(np.int64))


def test_big_pair_accuracy(gpu, oracle):
    """C5-style ribbon: 20k x 20k vs the oracle, 100k x 100k vs the analytic lambda."""
    a, b = lc.generators.ribbon_pair(10, 20000)
    want = oracle.link_direct(a, b)
    for mode in MODES:
        assert abs(gpu.link_direct(a, b, mode) - want) < RAW_TOL
    a, b = lc.generators.ribbon_pair(10, 100000)
    for mode in (_native.GAUSS_PHASE, _native.GAUSS_ATAN):
        assert abs(gpu.link_direct(a, b, mode) - 10.0) < RAW_TOL


def test_knit_tube_rows_sample(gpu, oracle):
    """C4 building block at reduced size: adjacent courses link -W; rows sample vs oracle."""
    m = lc.generators.knit_tube(courses=4, n=20000, W=100)
    mat = lc.compute_linking_matrix(m)
    assert mat.entries == ((0, 1, -100), (1, 2, -100), (2, 3, -100))
    a, b = (lp.control_points for lp in m.loops[:2])
    full = oracle.link_direct(a, b)
    assert abs(gpu.link_direct(a, b) - full) < RAW_TOL


def test_edge_cases(gpu):
    ex, ey, ez = np.eye(3)
    with pytest.raises(lc.ValidationError):
        lc.potential_link_search(lc.CurveModel([]))
    single = lc.CurveModel([lc.LoopGeometry.from_polyline(cases.circ(8, (0, 0, 0), ex, ey))])
    assert len(lc.potential_link_search(single)) == 0
    assert lc.compute_linking_matrix(single).entries == ()
    a = cases.circ(16, (0, 0, 0), ex, ey)
    b = cases.circ(16, (1.0, 0, 0), ez, ex)
    hopf = lc.CurveModel([lc.LoopGeometry.from_polyline(p) for p in (a, b)])
    assert lc.compute_linking_matrix(hopf, excluded={(1, 0)}).entries == ()
    assert lc.compute_linking_matrix(hopf).entries == ((0, 1, 1),)
    # NaN raw -> ValueError like round(nan)
    nan = a.copy()
    nan[3, 0] = np.nan
    with pytest.raises(ValueError):
        lc.compute_link(nan, b)
    # empty pair list through the batched seam
    raw, lk, flags = gpu.evaluate_pairs(np.concatenate([a, b]), np.array([0, 16, 32]), np.zeros((0, 2), np.int32))
    assert raw.shape == (0,)


@pytest.mark.parametrize("mode", MODES)
def test_degenerate_shared_vertices_vs_oracle(gpu, oracle, mode):
    """Coincident vertices (|r| = 0, w = 0): the phase fast path must fall back to the
    exact per-pair evaluation and agree with the reference's atan2(+-0, +-0) semantics."""
    ex, ey, ez = np.eye(3)
    a = cases.circ(24, (0, 0, 0), ex, ey)
    b = cases.circ(24, (1.0, 0, 0), ez, ex)
    b[5] = a[0]                                  # a shared vertex
    c = a.copy()
    c[3] = c[4]                                  # duplicate vertex inside one loop (zero-length segment)
    for x, y in ((a, b), (c, b), (a, a + 1e-300), (a, a)):
        want = oracle.link_direct(x, y)
        got = gpu.link_direct(x, y, mode)
        assert (np.isnan(want) and np.isnan(got)) or abs(got - want) < RAW_TOL, (want, got)


def test_env_mode_selection(monkeypatch):
    ex, ey, ez = np.eye(3)
    a = cases.circ(100, (0, 0, 0), ex, ey)
    b = cases.circ(100, (1.0, 0, 0), ez, ex)
    for name in ("phase", "atan", "ref"):
        monkeypatch.setenv("LINKCERT_GAUSS_MODE", name)
        assert lc.link_direct(a, b) == pytest.approx(1.0, abs=1e-12)
    monkeypatch.setenv("LINKCERT_GAUSS_MODE", "bogus")
    with pytest.raises(ValueError):
        lc.link_direct(a, b)


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    """The product path must fail loudly without the CUDA library (no oracle, no numpy fallback)."""
    monkeypatch.setattr(_native, "LIB_PATH", tmp_path / "missing.so")
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "_ctx", {})
    with pytest.raises(_native.NativeUnavailable):
        lc.link_direct(np.eye(3), np.eye(3) + 5)


def _pipeline_outcome(model, excluded=(), params=None):
    """(pairs, raw, lk, flags) bytes of the device pipeline, or the error it raises."""
    from paper_2106_12655_b200.certify import run_device_pipeline

    try:
        pairs, raw, lk, flags, ctx = run_device_pipeline(model, excluded, params)
        return ("ok", np.array(pairs).tobytes(), np.array(raw).tobytes(), np.array(lk).tobytes(),
                np.array(flags).tobytes()), ctx.last_run_fused()
    except (lc.DiscretizationError, lc.ValidationError) as e:
        return (type(e).__name__, getattr(e, "kind", None), tuple(getattr(e, "loops", ()) or ()), str(e)), None


def test_fused_matches_staged(monkeypatch, cert_models):
    """The fused single-sync pipeline and the staged one give bitwise-identical
    results and identical errors; the fused one runs wherever it applies."""
    ex, ey, ez = np.eye(3)
    runs = {name: (m, (), None) for name, m in cert_models.items()}
    for name, (_, after) in cases.edit_cases().items():
        runs["edit_" + name] = (after, (), None)
    for name, (m, _, kw) in cases.disc_error_cases().items():
        runs["disc_" + name] = (m, (), lc.DiscretizationParams(**kw))
    for name, m in cases.validation_cases().items():
        runs["val_" + name] = (m, (), None)
    a, b = cases.circ(16, (0, 0, 0), ex, ey), cases.circ(16, (1.0, 0, 0), ez, ex)
    hopf = lc.CurveModel([lc.LoopGeometry.from_polyline(p) for p in (a, b)])
    runs["hopf_excluded"] = (hopf, {(1, 0)}, None)
    fused_names = []
    for name, (m, excl, prm) in runs.items():
        monkeypatch.setenv("LINKCERT_FUSED", "0")
        staged, used = _pipeline_outcome(m, excl, prm)
        assert not used
        monkeypatch.setenv("LINKCERT_FUSED", "1")
        fused, used = _pipeline_outcome(m, excl, prm)
        assert fused == staged, name
        if not used:   # a first run past the item capacity falls back and sizes it
            fused, used = _pipeline_outcome(m, excl, prm)
            assert fused == staged, name
        if used:
            fused_names.append(name)
    # polyline models that need no refinement take the fused path
    for name in ("grid6", "unlinked200", "e4in1_32x32", "kusari_small", "hopf_excluded"):
        assert name in fused_names, (name, fused_names)


def test_fused_graph_replay_bitwise(monkeypatch):
    """Repeated runs of one model: plain fused run, capture, then graph replays —
    all bitwise equal to the staged path; a reallocation forces a recapture."""
    from paper_2106_12655_b200.certify import run_device_pipeline

    monkeypatch.setenv("LINKCERT_FUSED", "0")
    m = lc.generators.kusari_tube(n_around=12, rows=4, partial=5)
    want = [np.array(a).copy() for a in run_device_pipeline(m)[:4]]
    monkeypatch.setenv("LINKCERT_FUSED", "1")
    # a fresh context: the first fused run sizes every buffer on the fly
    *got, _ = run_device_pipeline(m, ctx=_native.Context())
    for a, b in zip(want, got):
        assert np.array_equal(a, np.asarray(b))
    paths = []
    for rep in range(5):
        if rep == 3:   # a bigger model on the same context reallocates buffers
            run_device_pipeline(lc.generators.kusari_tube(n_around=16, rows=6, partial=3))
        *got, ctx = run_device_pipeline(m)
        paths.append(ctx.last_run_fused())
        st = ctx.stage_times()   # without stage detail the graph records only the Gauss-stage events
        assert st["gauss"] > 0.0 and all(v is None for k, v in st.items() if k != "gauss")
        for a, b in zip(want, got):
            assert np.array_equal(a, np.asarray(b)) and np.asarray(b).dtype == a.dtype
    assert paths[0] >= 1 and 2 in paths, paths
    for rep in range(3):   # with detail (a caller asking for timings): every stage, replayed graphs too
        tm = {}
        *got, ctx = run_device_pipeline(m, timings=tm)
        assert all(v is not None and v >= 0.0 for v in ctx.stage_times().values())
        assert tm["kernel"] > 0.0 and tm["pls"] > 0.0
        for a, b in zip(want, got):
            assert np.array_equal(a, np.asarray(b))


def test_fused_pair_capacity_growth(monkeypatch, cert_models):
    """The pair capacity follows the largest pair count seen on a context: a model
    with more pairs than that overflows it once (staged fallback, same results),
    and the next fused run is sized for it."""
    from paper_2106_12655_b200.certify import run_device_pipeline

    big = cert_models["e4in1_32x32"]    # 2,945 pairs > the capacity a 6x6 grid leaves
    monkeypatch.setenv("LINKCERT_FUSED", "0")
    want = [np.array(a).copy() for a in run_device_pipeline(big)[:4]]
    monkeypatch.setenv("LINKCERT_FUSED", "1")
    ctx = _native.Context()
    run_device_pipeline(cert_models["grid6"], ctx=ctx)
    assert ctx.last_run_fused() == 1
    paths = []
    for _ in range(3):
        *got, _ = run_device_pipeline(big, ctx=ctx)
        paths.append(ctx.last_run_fused())
        for a, b in zip(want, got):
            assert np.array_equal(a, np.asarray(b))
    assert paths[0] == 0 and paths[1] >= 1, paths


@pytest.mark.parametrize("name", list(cases.validation_cases()))
def test_pipeline_validation_errors(golden, monkeypatch, name):
    """A chord PolylineLoop failure through the whole pipeline raises the reference's
    ValidationError on the fused path (read back with the run's status) and on the
    staged path alike."""
    g = golden["validation"][name]
    m = cases.validation_cases()[name]
    assert cases.fingerprint(m) == g["fingerprint"]
    assert [list(p) for p in lc.potential_link_search(m)] == g["pairs"]
    for fused in ("1", "0"):
        monkeypatch.setenv("LINKCERT_FUSED", fused)
        with pytest.raises(lc.ValidationError) as e:
            lc.compute_linking_matrix(m)
        assert str(e.value) == g["message"]
        assert _native.context().last_run_fused() == (1 if fused == "1" else 0)


class _DeviceArray:
    """Zero-copy torch view of a library-owned device buffer (__cuda_array_interface__)."""

    def __init__(self, ptr, n, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3}


def _mixed_model():
    """Kusari rings + knit courses of very different sizes: item costs vary ~60x."""
    k = lc.generators.kusari_tube(n_around=12, rows=4, partial=5)
    kv = k.snapshot()
    knit = lc.generators.knit_tube(courses=4, n=3000, W=10)
    kn = knit.snapshot()
    shift = np.array([200.0, 0.0, 0.0])
    verts = np.concatenate([kv.vertices(), kn.vertices() + shift])
    off = np.concatenate([kv.off, kn.off[1:] + kv.off[-1]])
    return lc.CurveModel.from_polyline_arrays(verts, off)


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_cost_balanced_shard_bounds(gpu, shards):
    """lc_shard_bounds: the ranges partition the items, and each rank's segment-pair
    cost is within one item of total / shards (north_star: split by estimated cost)."""
    from paper_2106_12655_b200.certify import run_device_pipeline

    m = _mixed_model()
    pairs, _, _, _, ctx = run_device_pipeline(m)
    pairs = np.array(pairs)
    ctx.prepare_gauss()
    b = ctx.shard_bounds(shards)
    assert b[0] == 0 and np.all(np.diff(b) >= 0)
    # per-item cost on the host from the pair sizes (items of a pair tile it exactly)
    _, voff = ctx.get_polylines()
    nseg = np.diff(voff)

    def tile(max_cl):
        items = []
        for i, j in pairs:
            g_rows, g_cols = int(nseg[j]), int(nseg[i])
            nb = -(-g_rows // 4)
            rbl = 0
            while (1 << rbl) < nb and rbl < 5:
                rbl += 1
            cs = 32 >> rbl
            cl = min(max(-(-g_cols // cs), 1), max_cl)
            rows_per, span = 4 << rbl, cs * cl
            for ir in range(-(-g_rows // rows_per)):
                for ic in range(-(-g_cols // span)):
                    items.append(min(rows_per, g_rows - ir * rows_per) * min(span, g_cols - ic * span))
        return np.array(items, dtype=np.int64)

    items = tile(2048)
    # Pipeline::retile_few_items: a model with loops the fused path does not take (> 256
    # segments) and fewer than 8 items per SM is tiled with shorter column strips
    import torch
    target = 8 * torch.cuda.get_device_properties(0).multi_processor_count
    if len(items) < target and nseg.max() > 256:
        max_cl, est = 2048, len(items)
        while est < target and max_cl > 16:
            est, max_cl = 2 * est, max_cl // 2
        items = tile(max_cl)
    assert b[-1] == len(items)
    total = items.sum()
    cum = np.concatenate([[0], np.cumsum(items)])
    assert total == int(np.sum(nseg[pairs[:, 0]] * nseg[pairs[:, 1]]))
    for r in range(shards):
        cost = cum[b[r + 1]] - cum[b[r]]
        assert abs(cost - total / shards) <= 2 * items.max(), (r, cost, total / shards)
    # the old equal-count split is far off on this model
    per = -(-len(items) // shards)
    counts = [cum[min(len(items), (r + 1) * per)] - cum[min(len(items), r * per)] for r in range(shards)]
    assert max(counts) - min(counts) > 2 * items.max()


@pytest.mark.parametrize("shards", [2, 3, 8])
def test_async_shards_allreduce_max_bitwise(shards):
    """The multi-GPU exchange emulated on one GPU: every shard's async fused run
    leaves its items in the partials buffer and -0.0 bits elsewhere; the int64
    MAX over the shards' buffers (what the NCCL all-reduce computes) handed to
    the pending run's lc_shard_finish gives bitwise the single-GPU results."""
    import torch

    from paper_2106_12655_b200.certify import excluded_keys, run_device_pipeline
    from paper_2106_12655_b200.pls import upload

    m = lc.generators.kusari_tube(n_around=12, rows=4, partial=5)
    want = [np.array(a).copy() for a in run_device_pipeline(m)[:4]]
    ctx = _native.Context()
    upload(m, ctx)
    prm = lc.DiscretizationParams()
    for rep in range(2):   # second round: graph replays
        bufs = []
        for r in range(shards):
            got = ctx.run_pipeline_shard_async(excluded_keys(()), m.xi, prm.epsilon, prm.max_passes,
                                               prm.max_subsegments, 0, r, shards)
            assert got is not None
            ptr, cap = got
            ctx.synchronize()
            bufs.append(torch.as_tensor(_DeviceArray(ptr, cap, "<i8"), device="cuda").clone())
        owned = torch.stack(bufs) != torch.iinfo(torch.int64).min
        assert int(owned.sum(dim=0).max()) <= 1            # every item has one owner
        combined = torch.stack(bufs).max(dim=0).values
        torch.as_tensor(_DeviceArray(ptr, cap, "<i8"), device="cuda").copy_(combined)
        torch.cuda.synchronize()
        assert ctx.shard_finish()
        got = ctx.result_views()
        for a, b in zip(want, got):
            assert np.array_equal(a, np.asarray(b)), (rep, shards)


def test_sharded_nccl_path_world1():
    """The multi-GPU code path (the library's own NCCL communicator: fused shard
    run + in-place MAX all-reduce on the library stream + fixed-order reduce, and
    the staged sharded path) end to end under torchrun at world size 1
    (LINKCERT_FORCE_SHARDED)."""
    import os
    import socket
    import subprocess
    import sys

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                          "--master-addr", "127.0.0.1", "--master-port", str(port),
                          os.path.join(root, "tools", "sharded_smoke.py")],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0 and "sharded smoke ok" in out.stdout, (out.stdout[-2000:], out.stderr[-2000:])


def _ring_soup(seed, count=400, n=24, size=12.0, spline=False):
    rng = np.random.default_rng(seed)
    th = 2 * np.pi * np.arange(n) / n
    loops = []
    for c in rng.uniform(0.0, size, size=(count, 3)):
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        v = np.cross(u, rng.normal(size=3))
        v /= np.linalg.norm(v)
        pts = c + np.outer(np.cos(th), u) + np.outer(np.sin(th), v)
        loops.append(lc.LoopGeometry.from_catmull_rom(pts) if spline else lc.LoopGeometry.from_polyline(pts))
    return lc.CurveModel(loops)


@pytest.mark.parametrize("spline", [False, True])
@pytest.mark.parametrize("seed,count,size", [(1, 400, 12.0), (2, 400, 12.0), (5, 150, 3.0)])
def test_random_ring_soup_vs_oracle(oracle, seed, count, size, spline):
    """Random overlapping rings (polyline or spline; near contacts need refinement
    passes; the dense soup has ~90 partners per PLS row, past the 16 row slots):
    the device certificate — PLS, discretization, Gauss sums, rounding — equals
    the oracle's, integers and pair lists exactly, raw sums within RAW_TOL."""
    from paper_2106_12655_b200.certify import run_device_pipeline

    m = _ring_soup(seed, count=count, size=size, spline=spline)
    coeffs, t, off = m.packed()
    want, pairs, raw = oracle.link_matrix(coeffs, t, off, m.xi)
    got = lc.compute_linking_matrix(m)
    assert np.array_equal(got.array, want)
    p2, r2, _, _, ctx = run_device_pipeline(m)
    assert np.array_equal(np.asarray(p2), pairs)
    assert np.max(np.abs(np.asarray(r2) - raw)) < RAW_TOL


def _edge_models():
    ex, ey, ez = np.eye(3)
    rng = np.random.default_rng(9)
    far = lc.CurveModel([lc.LoopGeometry.from_polyline(cases.circ(8, (0, 0, 0), ex, ey)),
                         lc.LoopGeometry.from_polyline(cases.circ(8, (50, 0, 0), ex, ey))])
    tris = []
    for c in rng.uniform(0, 4, size=(300, 3)):
        pts = c + rng.normal(size=(3, 3)) * 0.6
        tris.append(lc.LoopGeometry.from_polyline(pts))
    tri_soup = lc.CurveModel(tris)
    # chains of alternately oriented rings (a Hopf link between neighbours)
    shifted = lc.CurveModel([lc.LoopGeometry.from_polyline(
        cases.circ(32, (1e6 + 1.2 * k, 0, 0), ex, ey) if k % 2 else cases.circ(32, (1e6 + 1.2 * k, 0, 0), ez, ex))
        for k in range(6)])
    tiny = lc.CurveModel([lc.LoopGeometry.from_polyline(
        cases.circ(16, (1.2e-6 * k, 0, 0), ex, ey, radius=1e-6) if k % 2 else
        cases.circ(16, (1.2e-6 * k, 0, 0), ez, ex, radius=1e-6)) for k in range(4)])
    # loops of 256 and 257 segments: either side of the fused path's loop-length limit
    long_loops = {n: lc.CurveModel([lc.LoopGeometry.from_polyline(cases.circ(n, (0, 0, 0), ex, ey)),
                                    lc.LoopGeometry.from_polyline(cases.circ(n, (1.0, 0, 0), ez, ex))])
                  for n in (256, 257)}
    mixed = lc.CurveModel([lc.LoopGeometry.from_polyline(cases.circ(16, (0, 0, 0), ex, ey)),
                           lc.LoopGeometry.from_catmull_rom(cases.circ(12, (1.0, 0, 0), ez, ex))])
    return {"far": far, "tri_soup": tri_soup, "shifted_1e6": shifted, "tiny_1e-6": tiny,
            "loops_256": long_loops[256], "loops_257": long_loops[257], "mixed_poly_spline": mixed}


@pytest.mark.parametrize("name", list(_edge_models()))
def test_edge_models_vs_oracle(oracle, name):
    """Edge geometry through the whole device path (fused and staged) vs the oracle:
    no pairs, 3-segment loops, large offsets, tiny scales, the fused path's
    loop-length limit, polyline + spline mixes."""
    from paper_2106_12655_b200.certify import run_device_pipeline

    m = _edge_models()[name]
    coeffs, t, off = m.packed()
    want, pairs, raw = oracle.link_matrix(coeffs, t, off, m.xi)
    assert np.array_equal(lc.compute_linking_matrix(m).array, want)
    p2, r2, _, _, ctx = run_device_pipeline(m)
    assert np.array_equal(np.asarray(p2).reshape(-1, 2), pairs.reshape(-1, 2))
    if len(raw):
        assert np.max(np.abs(np.asarray(r2) - raw)) < RAW_TOL
