"""CPU tests of the host-side mirror of the reference API (no GPU compute).

Ported from the reference's own unit tests where they exercise host logic
(test_certify.py:27-137, test_pls.py:55-66, test_kernels.py:49-67,
test_discretize.py:126-132, test_geometry.py) plus the B200 additions:
packed-model layout, native digest and the vectorized verify diff.
"""

import numpy as np
import pytest

import cases
import paper_2106_12655_b200 as lc
from conftest import circle_points
from paper_2106_12655_b200 import _native
from paper_2106_12655_b200.certify import ABORTED, FAIL, PASS, diff_arrays
from paper_2106_12655_b200.geometry import compute_xi
from paper_2106_12655_b200.model_io import model_digest_python


# ------------------------------------------------------------ certificates

def test_serialize_parse_roundtrip_bytewise():
    m = lc.LinkMatrix(4, ((0, 1, 2), (1, 3, -1)), model_digest="abc", kernel_tag="ds:atan")
    data = lc.serialize_matrix(m)
    again = lc.parse_matrix(data)
    assert again == m
    assert lc.serialize_matrix(again) == data
    assert data == b'{"digest":"abc","entries":[[0,1,2],[1,3,-1]],"kernel":"ds:atan","num_loops":4}'


def test_matrix_invariants():
    with pytest.raises(lc.ValidationError):
        lc.LinkMatrix(3, ((1, 2, 1), (0, 1, 1)))
    with pytest.raises(lc.ValidationError):
        lc.LinkMatrix(3, ((0, 1, 1), (0, 1, 2)))
    with pytest.raises(lc.ValidationError):
        lc.LinkMatrix(3, ((0, 1, 0),))
    with pytest.raises(lc.ValidationError):
        lc.LinkMatrix(3, ((1, 1, 2),))
    with pytest.raises(lc.ValidationError):
        lc.LinkMatrix(2, ((0, 5, 1),))
    m = lc.LinkMatrix(3, ((0, 2, -4),))
    assert m[(2, 0)] == -4
    assert m[(0, 1)] == 0
    empty = lc.LinkMatrix(5)
    assert empty.entries == ()
    assert lc.parse_matrix(lc.serialize_matrix(empty)) == empty
    with pytest.raises(AttributeError):
        m.num_loops = 7


def test_parse_errors():
    with pytest.raises(lc.ParseError):
        lc.parse_matrix(b"{not json")
    with pytest.raises(lc.ParseError):
        lc.parse_matrix(b'{"num_loops": 2}')
    with pytest.raises(lc.ParseError):
        lc.parse_matrix(b'{"num_loops":2,"digest":"","kernel":"","entries":[[1,0,1]]}')


def test_diff_matrices_classification():
    a = lc.LinkMatrix(4, ((0, 1, 1), (1, 2, 2)))
    b = lc.LinkMatrix(4, ((1, 2, 3), (2, 3, 1)))
    report = lc.diff_matrices(a, b)
    assert report.status == FAIL
    assert report.destroyed == [(0, 1)]
    assert report.created == [(2, 3)]
    assert report.changed == [(1, 2)]
    assert lc.diff_matrices(a, a).status == PASS
    assert lc.diff_matrices(a, lc.LinkMatrix(9)).status == FAIL
    assert report.failing_pairs() == [(0, 1), (1, 2), (2, 3)]
    assert report.as_dict()["first_failure"] is None


def _random_case(rng, L=60):
    cand = sorted({tuple(sorted(rng.choice(L, 2, replace=False).tolist())) for _ in range(200)})
    pairs = np.array(cand, dtype=np.int32)
    lk = rng.integers(-2, 3, size=len(pairs))
    ref_pairs = sorted({tuple(sorted(rng.choice(L, 2, replace=False).tolist())) for _ in range(120)})
    ref = [(i, j, int(v)) for (i, j), v in zip(ref_pairs, rng.integers(-2, 3, size=len(ref_pairs))) if v != 0]
    return pairs, lk, ref


def _reference_verify(pairs, lk, ref, early_exit):
    """Direct restatement of certify.verify's ordering / diff (certify.py:194-221)."""
    refd = {(i, j): v for i, j, v in ref}
    values_all = {tuple(p): int(v) for p, v in zip(pairs.tolist(), lk.tolist())}
    candidate = set(values_all)
    ordering = sorted(refd) + sorted(candidate - set(refd))
    if early_exit:
        values = {}
        for pair in ordering:
            lam = values_all[pair] if pair in candidate else 0
            values[pair] = lam
            if lam != refd.get(pair, 0):
                d = _diff_dicts({p: refd[p] for p in values if p in refd}, values)
                return ABORTED, d, pair
        return PASS, ([], [], []), None
    values = {p: values_all[p] for p in ordering if p in candidate}
    for p in ordering:
        values.setdefault(p, 0)
    d = _diff_dicts(refd, values)
    return (FAIL if any(d) else PASS), d, None


def _diff_dicts(ref, computed):
    out = ([], [], [])
    for pair in sorted(set(ref) | set(computed)):
        w, g = ref.get(pair, 0), computed.get(pair, 0)
        if w == g:
            continue
        out[0 if (w and not g) else 1 if (g and not w) else 2].append(pair)
    return out


@pytest.mark.parametrize("seed", range(30))
@pytest.mark.parametrize("early_exit", [False, True])
def test_vectorized_verify_diff_matches_reference_logic(seed, early_exit):
    rng = np.random.default_rng(seed)
    pairs, lk, ref = _random_case(rng)
    if seed % 5 == 0:          # a passing case
        ref = [(int(i), int(j), int(v)) for (i, j), v in zip(pairs.tolist(), lk.tolist()) if v != 0]
    raw = lk.astype(float) + 1e-12
    flags = np.zeros(len(pairs), dtype=np.uint8)
    ref_arr = np.array(ref, dtype=np.int64).reshape(-1, 3)
    rep = diff_arrays(ref_arr, pairs, raw, lk, flags, early_exit)
    status, (d, c, ch), first = _reference_verify(pairs, lk, ref, early_exit)
    assert rep.status == status
    assert (rep.destroyed, rep.created, rep.changed) == (d, c, ch)
    assert rep.first_failure == first


def test_verify_diff_raises_like_round_on_nan():
    pairs = np.array([[0, 1], [1, 2]], dtype=np.int32)
    lk = np.array([1, 0])
    raw = np.array([1.0, np.nan])
    flags = np.array([0, _native.FLAG_NAN], dtype=np.uint8)
    ref = np.array([[0, 1, 1]], dtype=np.int64)
    with pytest.raises(ValueError):
        diff_arrays(ref, pairs, raw, lk, flags, False)
    # early exit stops before the NaN pair when an earlier pair already fails
    ref2 = np.array([[0, 1, 5]], dtype=np.int64)
    rep = diff_arrays(ref2, pairs, raw, lk, flags, True)
    assert rep.status == ABORTED and rep.first_failure == (0, 1)


# ---------------------------------------------------------- data model

def test_pairlist_invariants():
    pl = lc.PairList(((2, 3), (0, 1), (2, 3)))
    assert pl.pairs == ((0, 1), (2, 3))
    assert len(pl) == 2
    assert pl.loops_involved() == {0, 1, 2, 3}
    with pytest.raises(lc.ValidationError):
        lc.PairList(((3, 2),))
    assert lc.PairList((), excluded={(5, 1)}).excluded == frozenset({(1, 5)})
    assert list(pl) == [(0, 1), (2, 3)]


def test_kernel_choice():
    assert lc.KernelChoice(method="ds", ds_variant="anglesum").tag == "ds:anglesum"
    assert lc.KernelChoice(method="bh", bh=lc.BarnesHutParams(order="dipole")).tag == "bh:dipole"
    assert lc.KernelChoice(method="cc").tag == "cc"
    with pytest.raises(ValueError):
        lc.KernelChoice(method="fmm")
    with pytest.raises(ValueError):
        lc.KernelChoice(ds_variant="simpson")
    from paper_2106_12655_b200.kernels import pair_choice

    base = lc.KernelChoice(method="cc", cc=lc.CrossingParams(seed=7))
    seeds = {pair_choice(base, i, j).cc.seed for i in range(5) for j in range(i + 1, 6)}
    assert len(seeds) == 15
    with pytest.raises(NotImplementedError):
        lc.compute_link(np.eye(3), np.eye(3), lc.KernelChoice(method="cc"))


def test_discretization_params_validation():
    with pytest.raises(ValueError):
        lc.DiscretizationParams(epsilon=0.0)
    with pytest.raises(ValueError):
        lc.DiscretizationParams(max_passes=0)
    with pytest.raises(ValueError):
        lc.DiscretizationParams(max_subsegments=0)


def test_failure_mapping_messages():
    from paper_2106_12655_b200.discretize import raise_for_failure

    p = lc.DiscretizationParams(max_passes=7, max_subsegments=9)
    cases_ = [
        (_native.DiscretizeFailure(_native.DISC_ZERO_LENGTH, 0, [3]), "ZeroLengthInput", (3,),
         "Input has zero-length segments."),
        (_native.DiscretizeFailure(_native.DISC_CURVES_INTERSECT, 0, [1, 2]), "CurvesIntersect", (1, 2),
         "Curves 1 and 2 intersect."),
        (_native.DiscretizeFailure(_native.DISC_SUBSEG_BUDGET, 0, [4]), "PassLimitExceeded", (4,),
         "loop 4 exceeded the 9 subsegment refinement budget"),
        (_native.DiscretizeFailure(_native.DISC_PASS_BUDGET, 0, [0, 1]), "PassLimitExceeded", (0, 1),
         "refinement did not settle within 7 passes"),
    ]
    for fail, kind, loops, msg in cases_:
        with pytest.raises(lc.DiscretizationError) as e:
            raise_for_failure(fail, p)
        assert (e.value.kind, e.value.loops, str(e.value)) == (kind, loops, msg)
    with pytest.raises(lc.ValidationError, match="zero-length segment"):
        raise_for_failure(_native.DiscretizeFailure(_native.DISC_INVALID_POLYLINE, 3, [2]), p)


def test_loop_and_polyline_validation():
    pts = circle_points(8)
    with pytest.raises(lc.ValidationError):
        lc.LoopGeometry.from_polyline(pts[:, :2])
    bad = pts.copy()
    bad[0, 0] = np.nan
    with pytest.raises(lc.ValidationError):
        lc.LoopGeometry.from_polyline(bad)
    with pytest.raises(lc.ValidationError):
        lc.LoopGeometry(np.zeros((2, 4, 3)))
    gap = np.zeros((3, 4, 3))
    gap[:, 0] = pts[:3]
    gap[:, 1] = 0.5 * (np.roll(pts[:3], -1, axis=0) - pts[:3])
    with pytest.raises(lc.ValidationError):
        lc.LoopGeometry(gap)
    with pytest.raises(lc.ValidationError):
        lc.PolylineLoop(pts[:2])
    with pytest.raises(lc.ValidationError):
        lc.PolylineLoop(np.vstack([pts, pts[-1:]]))
    assert len(lc.PolylineLoop(pts)) == 8
    loop = lc.LoopGeometry.from_catmull_rom(pts)
    assert len(loop) == 8
    assert np.allclose(loop.start_points(), pts)
    assert np.allclose(loop.end_points(), np.roll(pts, -1, axis=0))
    with pytest.raises(lc.ValidationError):
        lc.LoopGeometry.from_catmull_rom(pts[:3])


def test_bulk_constructor_equals_per_loop_construction():
    rng = np.random.default_rng(11)
    loops = [circle_points(int(n), center=rng.normal(size=3) * 5, radius=float(r))
             for n, r in zip(rng.integers(3, 40, 30), rng.uniform(0.5, 3, 30))]
    off = np.concatenate([[0], np.cumsum([len(x) for x in loops])])
    bulk = lc.CurveModel.from_polyline_arrays(np.concatenate(loops), off)
    slow = lc.CurveModel([lc.LoopGeometry.from_polyline(p) for p in loops])
    assert bulk.xi == slow.xi == compute_xi(slow.loops)
    for a, b in zip(bulk.packed(), slow.packed()):
        assert np.array_equal(a, b)
    for la, lb in zip(bulk.loops, slow.loops):
        assert np.array_equal(la.control_points, lb.control_points)
        assert np.array_equal(la.coeffs, lb.coeffs)


def test_generators_reproduce_golden_inputs(golden):
    for name, m in cases.link_cases().items():
        assert cases.fingerprint(m) == golden["links"][name]["fingerprint"], name
    for name, m in cases.cert_models().items():
        assert cases.fingerprint(m) == golden["certs"][name]["fingerprint"], name
        assert m.xi == golden["certs"][name]["xi"], name


def test_native_digest_matches_reference(golden):
    for name, m in cases.cert_models().items():
        assert lc.model_digest(m) == golden["certs"][name]["digest"], name
        assert model_digest_python(m) == golden["certs"][name]["digest"], name
    for name, (_, after) in cases.edit_cases().items():
        assert lc.model_digest(after) == golden["verify"][name]["after_digest"], name


def test_digest_cubics_and_open_loops():
    """Spline (cubics branch), non-unit domains and open polylines serialize like json.dumps."""
    m, _ = lc.generators.perturbed_random_link(seed=1, n=40, spline=True)
    assert lc.model_digest(m) == model_digest_python(m)
    seg = lc.CubicSegment.straight([0.0, 0.0, 0.0], [1.0, 2.0, 3.5])
    half = lc.CubicSegment(seg.coeffs, 0.25, 0.75)
    loop = lc.LoopGeometry.from_segments([half, lc.CubicSegment.straight(half.end, [0.1, -1e-7, 1e17]),
                                          lc.CubicSegment.straight([0.1, -1e-7, 1e17], half.start)])
    m2 = lc.CurveModel([loop, lc.LoopGeometry.from_polyline(circle_points(5) * 1e-5, closed=False)])
    assert lc.model_digest(m2) == model_digest_python(m2)


def test_streamed_snapshot_digest():
    """verify / compute_linking_matrix start the digest after the snapshot's first
    piece of loops (lc_model_digest_polylines_stream): the same digest as the
    finished snapshot's, the same snapshot arrays; a loop that is not a closed
    polyline past the first piece aborts the stream and the regular digest runs."""
    from paper_2106_12655_b200 import certify, workloads
    from paper_2106_12655_b200.geometry import ModelSnapshot

    v, off = workloads.kusari_tube_vertices(rows=40, n_around=60)
    loops = [lc.LoopGeometry.from_polyline(v[off[k]:off[k + 1]]) for k in range(len(off) - 1)]
    assert len(loops) > 2 * 1024
    m = lc.CurveModel(list(loops))
    want = model_digest_python(m)
    snap, digest_of = certify.snapshot_and_digest(m, None)
    assert snap.ready is not None and snap.ready[0] == len(loops)        # it was streamed
    assert digest_of() == want == lc.model_digest(lc.CurveModel(list(loops)))
    plain = ModelSnapshot(loops, 0)
    assert np.array_equal(snap.off, plain.off) and np.array_equal(snap.vptrs, plain.vptrs)
    assert np.array_equal(snap.vertices(), v)
    spline = lc.LoopGeometry.from_catmull_rom(v[off[3]:off[4]])
    mixed = lc.CurveModel(loops[:1500] + [spline] + loops[1500:2500])
    snap, digest_of = certify.snapshot_and_digest(mixed, None)
    assert not snap.poly and snap.ready[0] == -1                          # aborted after the first piece
    assert digest_of() == model_digest_python(mixed)
    snap, digest_of = certify.snapshot_and_digest(mixed, None)            # cached snapshot: regular digest
    assert digest_of() == model_digest_python(mixed)


# ------------------------------------------------------------- sharding

def _gloo_comm_worker(rank, world, port, q):
    """ensure_comm + digest_on_rank0 host logic over gloo: one unique id and one
    digest (rank 0's) reach every rank; a digest error reaches every rank too."""
    import os

    import torch.distributed as dist

    from paper_2106_12655_b200 import _native, certify

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _native.comm_unique_id = lambda: bytes([7]) * 128      # no NCCL on the CPU box: the exchange is the test

    class Ctx:
        comm = None

        def comm_init(self, uid, w, r):
            self.comm = (w, r)
            self.uid = uid

    ctx = Ctx()
    certify.ensure_comm(ctx, dist)
    certify.ensure_comm(ctx, dist)                          # idempotent: no second exchange
    calls = []
    certify._digest_async = lambda model, snap, nthreads=0: calls.append(nthreads) or _Done("d" + str(model))
    got = certify.digest_on_rank0("M", None, dist)()
    certify._digest_async = lambda model, snap, nthreads=0: _Done(exc=ValueError("cannot serialize"))
    try:
        certify.digest_on_rank0("M", None, dist)()
        err = None
    except ValueError as exc:
        err = str(exc)
    q.put((rank, ctx.comm == (world, rank) and ctx.uid == bytes([7]) * 128, got, len(calls), err))
    dist.destroy_process_group()


class _Done:
    def __init__(self, val=None, exc=None):
        self.val, self.exc = val, exc

    def result(self):
        if self.exc is not None:
            raise self.exc
        return self.val


@pytest.mark.parametrize("world", [2, 3])
def test_multirank_comm_and_digest_exchange(world):
    """world_size > 1 host logic on CPU (gloo): the library communicator's unique id
    and the model digest are made on rank 0 only and received by every rank."""
    import multiprocessing as mp
    import random

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_gloo_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert [r[0] for r in res] == list(range(world))
    assert all(r[1] and r[2] == "dM" and r[4] == "cannot serialize" for r in res)
    assert [r[3] for r in res] == [1] + [0] * (world - 1)      # only rank 0 hashed


def _gloo_max_worker(rank, world, port, n_items, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    vals = np.random.default_rng(7).normal(size=n_items) * 10.0 ** np.random.default_rng(8).integers(-300, 300, n_items)
    vals[::5] = -0.0
    vals[1::7] = 0.0
    vals[2::11] = np.inf
    vals[3::13] = -np.inf
    vals[4::17] = 5e-324                            # subnormal
    bits = vals.view(np.int64).copy()
    bits[6::19] = 0x7FF8DEADBEEF0001                # NaN with a payload
    cap = -(-n_items // world) * world + 3          # capacity > n_items, like the library buffer
    buf = torch.full((cap,), torch.iinfo(torch.int64).min, dtype=torch.int64)   # bits of -0.0
    bounds = np.linspace(0, n_items, world + 1).astype(np.int64)   # any partition (the library's is by cost)
    b, e = bounds[rank], bounds[rank + 1]
    buf[b:e] = torch.from_numpy(bits[b:e])          # the items this rank's Gauss slice wrote
    dist.all_reduce(buf, op=dist.ReduceOp.MAX)      # what lc_run_pipeline_sharded enqueues (NCCL)
    ok = bool(np.array_equal(buf.numpy()[:n_items], bits))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_items", [(2, 18749), (3, 1000)])
def test_multirank_max_allreduce_assembles_bits(world, n_items):
    """The fused multi-GPU exchange on CPU (gloo): items of other ranks hold the
    bits of -0.0 (INT64_MIN), so an int64 MAX all-reduce returns every item's bit
    pattern unchanged (signed zeros, infinities, subnormals, NaN payloads)."""
    import multiprocessing as mp
    import random

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    procs = [ctx.Process(target=_gloo_max_worker, args=(r, world, port, n_items, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, True) for r in range(world)]


def test_snapshot_tracks_the_loops():
    """The model snapshot (what verify uploads and hashes) is reused only while the
    loop list holds the same objects and no loop had an attribute reassigned."""
    import numpy as np

    from paper_2106_12655_b200 import generators as gen

    m = gen.kusari_tube(n_around=12, rows=4, partial=5)
    snap = m.snapshot()
    assert snap.poly and m.snapshot() is snap
    assert np.array_equal(snap.vertices(), np.concatenate([lp.control_points for lp in m.loops]))
    m.loops.append(m.loops[0])                      # list changed -> new snapshot
    s2 = m.snapshot()
    assert s2 is not snap and s2.off[-1] == snap.off[-1] + len(m.loops[0])
    assert np.array_equal(s2.packed()[0][:len(snap.packed()[0])], snap.packed()[0])
    m.loops.pop()
    s3 = m.snapshot()
    fresh = lc.CurveModel(list(m.loops), xi=m.xi)   # a fresh model of the same loops
    assert fresh.snapshot() is not s3 and np.array_equal(fresh.snapshot().vptrs, s3.vptrs)


def test_loop_arrays_are_owned_and_read_only():
    """an in-place edit cannot leave a cached snapshot stale —
    the loop owns read-only copies; reassignment invalidates the snapshot and
    drops the vertex-only fast path for that loop."""
    import numpy as np

    pts = circle_points(16)
    loop = lc.LoopGeometry.from_polyline(pts)
    pts[0, 0] += 1.0                                # the caller's array is not aliased
    assert loop.control_points[0, 0] != pts[0, 0]
    with pytest.raises(ValueError):
        loop.coeffs[0, 0, 2] += 3.0
    with pytest.raises(ValueError):
        loop.control_points[0] = 0.0
    m = lc.CurveModel([loop, lc.LoopGeometry.from_polyline(circle_points(16, center=(5, 0, 0)))])
    s1 = m.snapshot()
    assert s1.poly
    c = loop.coeffs.copy()
    c[:, 0, 2] += 3.0
    loop.coeffs = c                                  # reassignment: tracked
    s2 = m.snapshot()
    assert s2 is not s1 and not s2.poly
    assert np.array_equal(s2.packed()[0][:16], c)
    assert m.snapshot() is s2                        # and cached again


def test_snapshot_poly_only_for_closed_from_polyline_loops():
    import numpy as np

    closed = lc.LoopGeometry.from_polyline(circle_points(8))
    generic = lc.LoopGeometry(closed.coeffs, closed.t)          # polyline-shaped, but generic
    assert lc.CurveModel([closed, closed]).snapshot().poly
    assert not lc.CurveModel([closed, generic]).snapshot().poly
    opened = lc.LoopGeometry.from_polyline(circle_points(8), closed=False)
    assert not lc.CurveModel([closed, opened]).snapshot().poly
    a, b = lc.CurveModel([closed, generic]).packed(), lc.CurveModel([closed, closed]).packed()
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
