"""Certificates, verification and diffing — drop-in for linkcert.certify.

Reference: linkcert/certify.py:21-250.  The whole numeric path of
compute_linking_matrix / verify — potential link search, discretization,
Gauss sums and rounding — runs on the GPU as one device-resident pipeline
(one upload of the packed model, results back as arrays); the host only
diffs integer arrays.  Early-exit verification computes every candidate
pair on the device and then replays the reference's evaluation order on
the host, which yields the identical report because the per-pair integers
are identical.

Multi-GPU: when torch.distributed is initialized with world_size > 1 (NCCL),
every rank runs the pipeline with the Gauss kernel restricted to its
cost-balanced range of the work items (computed on the device); the per-item
partials are exchanged over the library's own NCCL communicator (an in-place
int64 MAX all-reduce enqueued behind the kernels) and every rank reduces them
in fixed order, so raw sums are bitwise identical for any number of ranks.
torch.distributed only carries the communicator's unique id and the model
digest, which rank 0 alone computes.
"""

from __future__ import annotations

import json
import os
import time
import warnings

import numpy as np

from . import _native
from .direct import ds_mode, gauss_mode
from .discretize import DiscretizationParams, raise_for_failure, split_polylines
from .geometry import CurveModel, ValidationError
from . import barneshut
from .kernels import (BARNES_HUT, AmbiguousLinkError, KernelChoice, ROUNDING_THRESHOLD, require_ds,
                      require_gpu_kernel)
from .model_io import ParseError, model_digest
from .pls import PairList, excluded_keys, upload

PASS = "Pass"
FAIL = "Fail"
ABORTED = "Aborted"


class LinkMatrix:
    """Sparse strictly-upper-triangular integer linking matrix (certify.py:27-53).

    Stores entries as an int64 (E, 3) array; the tuple view is built lazily.
    Equality ignores `diagnostics`, as in the reference.
    """

    __slots__ = ("num_loops", "_arr", "_entries", "model_digest", "kernel_tag", "diagnostics")

    def __init__(self, num_loops, entries=(), model_digest="", kernel_tag="", diagnostics=None):
        rows = [(int(i), int(j), int(lam)) for i, j, lam in entries]
        arr = np.asarray(rows, dtype=np.int64).reshape(-1, 3)
        if rows != sorted(rows) or len({r[:2] for r in rows}) != len(rows):
            raise ValidationError("entries must be sorted and unique")
        for i, j, lam in rows:
            if not 0 <= i < j < num_loops:
                raise ValidationError(f"entry ({i}, {j}) out of triangular range")
            if lam == 0:
                raise ValidationError("zero entries must not be stored")
        self._init(int(num_loops), arr, tuple(rows), model_digest, kernel_tag, diagnostics)

    def _init(self, num_loops, arr, entries, digest, tag, diagnostics):
        object.__setattr__(self, "num_loops", num_loops)
        object.__setattr__(self, "_arr", arr)
        object.__setattr__(self, "_entries", entries)
        object.__setattr__(self, "model_digest", digest)
        object.__setattr__(self, "kernel_tag", tag)
        object.__setattr__(self, "diagnostics", {} if diagnostics is None else diagnostics)

    @classmethod
    def _from_array(cls, num_loops, arr, model_digest="", kernel_tag="", diagnostics=None):
        """Trusted constructor: arr (E, 3) int64 already sorted, unique, i<j, lam != 0."""
        self = cls.__new__(cls)
        self._init(int(num_loops), np.ascontiguousarray(arr, dtype=np.int64).reshape(-1, 3), None,
                   model_digest, kernel_tag, diagnostics)
        return self

    def __setattr__(self, name, value):
        raise AttributeError(f"cannot assign to field {name!r}")   # frozen, like the dataclass

    @property
    def entries(self):
        if self._entries is None:
            object.__setattr__(self, "_entries", tuple(map(tuple, self._arr.tolist())))
        return self._entries

    @property
    def array(self):
        return self._arr

    def __eq__(self, other):
        if other.__class__ is not self.__class__:
            return NotImplemented
        return (self.num_loops == other.num_loops and np.array_equal(self._arr, other._arr)
                and self.model_digest == other.model_digest and self.kernel_tag == other.kernel_tag)

    def __hash__(self):
        return hash((self.num_loops, self.entries, self.model_digest, self.kernel_tag))

    def __repr__(self):
        return (f"LinkMatrix(num_loops={self.num_loops}, entries={self.entries!r}, "
                f"model_digest={self.model_digest!r}, kernel_tag={self.kernel_tag!r})")

    def as_dict(self):
        return {(i, j): lam for i, j, lam in self.entries}

    def __getitem__(self, pair):
        i, j = min(pair), max(pair)
        keys = (self._arr[:, 0] << 32) | self._arr[:, 1]
        k = (i << 32) | j
        pos = int(np.searchsorted(keys, k))
        return int(self._arr[pos, 2]) if pos < len(keys) and keys[pos] == k else 0


class VerificationReport:
    """certify.py:56-80."""

    def __init__(self, status, destroyed=None, created=None, changed=None, first_failure=None, message=""):
        self.status = status
        self.destroyed = [] if destroyed is None else destroyed
        self.created = [] if created is None else created
        self.changed = [] if changed is None else changed
        self.first_failure = first_failure
        self.message = message

    def __eq__(self, other):
        if other.__class__ is not self.__class__:
            return NotImplemented
        return self.as_dict() == other.as_dict()

    def __repr__(self):
        return (f"VerificationReport(status={self.status!r}, destroyed={self.destroyed!r}, created={self.created!r}, "
                f"changed={self.changed!r}, first_failure={self.first_failure!r}, message={self.message!r})")

    @property
    def ok(self):
        return self.status == PASS

    def failing_pairs(self):
        return sorted(set(self.destroyed) | set(self.created) | set(self.changed))

    def as_dict(self):
        return {
            "status": self.status,
            "destroyed": [list(p) for p in self.destroyed],
            "created": [list(p) for p in self.created],
            "changed": [list(p) for p in self.changed],
            "first_failure": list(self.first_failure) if self.first_failure else None,
            "message": self.message,
        }


def serialize_matrix(m: LinkMatrix) -> bytes:
    """Canonical JSON bytes; byte equality is matrix equality (certify.py:83-91)."""
    doc = {
        "num_loops": m.num_loops,
        "digest": m.model_digest,
        "kernel": m.kernel_tag,
        "entries": m.array.tolist(),
    }
    return json.dumps(doc, sort_keys=True, separators=(",", ":")).encode()


def parse_matrix(data: bytes) -> LinkMatrix:
    """certify.py:94-105."""
    try:
        doc = json.loads(data)
        return LinkMatrix(
            num_loops=int(doc["num_loops"]),
            entries=tuple((int(i), int(j), int(lam)) for i, j, lam in doc["entries"]),
            model_digest=str(doc["digest"]),
            kernel_tag=str(doc["kernel"]),
        )
    except (ValueError, KeyError, TypeError) as exc:
        raise ParseError(f"bad certificate: {exc}") from exc


# ----------------------------------------------------------------- device path

def _pair_keys(arr):
    arr = np.asarray(arr, dtype=np.int64).reshape(-1, 2)
    return (arr[:, 0] << 32) | arr[:, 1]


def _dist():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover - torch is part of the image
        return None
    if dist.is_available() and dist.is_initialized():
        # LINKCERT_FORCE_SHARDED=1 exercises the sharded code path at world size 1 (tests)
        if dist.get_world_size() > 1 or os.environ.get("LINKCERT_FORCE_SHARDED") == "1":
            return dist
    return None


def ensure_comm(ctx, dist):
    """The library's own NCCL communicator for this process group (created once):
    rank 0 makes the unique id, torch.distributed only carries those 128 bytes."""
    world, rank = dist.get_world_size(), dist.get_rank()
    if getattr(ctx, "comm", None) == (world, rank):
        return
    obj = [_native.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx.comm_init(obj[0], world, rank)


def snapshot_and_digest(model, dist):
    """(model.snapshot(), digest_on_rank0's callable).  Single process, fresh
    snapshot of closed polylines: the digest starts on its helper thread after
    the snapshot's first piece of loops (a streamed digest), so the ~1 ms walk
    over the loops overlaps the hash instead of preceding it."""
    if dist is not None:
        snap = model.snapshot()
        return snap, digest_on_rank0(model, snap, dist)
    started = []

    def start(sn):
        started.append(_digest_pool_submit(_native.model_digest_polylines_stream, sn.vptrs, sn.off, sn.ready))

    snap = model.snapshot(on_start=start)
    if not started:
        return snap, digest_on_rank0(model, snap, None)
    fut = started[0]
    if not snap.poly:   # the stream was aborted (a loop is not a closed polyline): the regular digest
        fut = _digest_async(model, snap)

    def result():
        try:
            digest = fut.result()
        except _native.DigestAborted:   # (not reached: an aborted stream is replaced above)
            digest = model_digest(model, snap)
        if digest is None:
            raise ValidationError("cannot serialize non-finite coordinate")
        return digest

    return snap, result


def digest_on_rank0(model, snapshot, dist):
    """model_digest computed once per job: rank 0 hashes (helper thread, overlapped
    with the GPU), the other ranks receive the string.  Returns a callable giving
    the digest (or raising the digest's error) on every rank."""
    if dist is None or dist.get_rank() == 0:
        world = 1 if dist is None else dist.get_world_size()
        fut = _digest_async(model, snapshot, nthreads=0 if world == 1 else max(2, (os.cpu_count() or 2) - world))
    else:
        fut = None

    def result():
        if dist is None:
            return fut.result()
        obj = [None]
        if fut is not None:
            try:
                obj[0] = ("ok", fut.result())
            except Exception as exc:  # noqa: BLE001 - re-raised on every rank below
                obj[0] = ("err", exc)
        dist.broadcast_object_list(obj, src=0)
        kind, val = obj[0]
        if kind == "err":
            raise val
        return val

    return result


def device_step(ctx, xi, excl_keys, params, mode=None, timings=None):
    """One pass of the hot path over the model resident on `ctx`:
    PLS -> discretize -> Gauss sum -> rounding.  Under torch.distributed (NCCL,
    world > 1) every rank evaluates its cost-balanced share of the work items
    and the library exchanges the partials over its own NCCL communicator.
    Returns (pairs int32 (P,2), raw, lk, flags) views in pinned host memory."""
    mode = gauss_mode() if mode is None else mode
    dist = _dist()
    args = (excl_keys, xi, params.epsilon, params.max_passes, params.max_subsegments, mode)
    if dist is not None and dist.get_backend() != "nccl":
        raise _native.NativeUnavailable("the multi-GPU path needs the NCCL backend on CUDA devices")
    ctx.set_stage_detail(timings is not None)   # every stage event only when the caller wants the stages
    try:
        if dist is None:
            ctx.run_pipeline(*args)          # one C-ABI call for the whole device path
        else:
            ensure_comm(ctx, dist)
            ctx.run_pipeline_sharded(*args)
    except _native.DiscretizeFailure as fail:
        raise_for_failure(fail, params)
    pairs, raw, lk, flags = ctx.result_views()   # pinned, valid until the next pipeline call
    if timings is not None:
        st = ctx.stage_times()
        timings["pls"] = timings.get("upload", 0.0) + 1e-3 * st["pls"]
        timings["discretize"] = 1e-3 * st["discretize"]
        timings["kernel"] = 1e-3 * (st["gauss"] + st["reduce"])
    return pairs, raw, lk, flags


def run_device_pipeline(model: CurveModel, excluded=(), params=None, timings=None, ctx=None, snapshot=None,
                        mode=None):
    """Upload the model snapshot, then device_step.  Returns (pairs, raw, lk, flags, ctx)."""
    params = params or DiscretizationParams()
    ctx = ctx or _native.context()
    with ctx.session:
        t0 = time.perf_counter()
        upload(model, ctx, snapshot)
        if timings is not None:
            timings["upload"] = time.perf_counter() - t0
        pairs, raw, lk, flags = device_step(ctx, model.xi, excluded_keys(excluded), params, mode=mode,
                                            timings=timings)
        if timings is not None:
            timings.pop("upload", None)
    return pairs, raw, lk, flags, ctx


_digest_pool = None


def _digest_pool_submit(fn, *args):
    global _digest_pool
    if _digest_pool is None:
        from concurrent.futures import ThreadPoolExecutor

        _digest_pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="linkcert-digest")
    return _digest_pool.submit(fn, *args)


def _digest_async(model, snapshot=None, nthreads=0):
    """model_digest on a helper thread (native, GIL released) to overlap it with the GPU."""
    return _digest_pool_submit(model_digest, model, snapshot, nthreads)


def _raise_for_flags(raw, flags, order=None):
    """Reproduce round()'s ValueError on NaN / the ambiguity rule, first offending pair first."""
    bad = np.nonzero(flags if order is None else flags[order])[0]
    if not len(bad):
        return
    k = int(bad[0]) if order is None else int(order[bad[0]])
    if flags[k] & _native.FLAG_NAN:
        raise ValueError("cannot convert float NaN to integer")
    raise AmbiguousLinkError(f"raw linking value {raw[k]!r} is ambiguous (> {ROUNDING_THRESHOLD} from an integer)")


def _evaluate_pairs(polylines, pair_items, choice, threads, diagnostics):
    """Integer link per (i, j) in one batched GPU call (certify.py:108-127)."""
    require_ds(choice or KernelChoice())
    if not pair_items:
        return {}
    counts = np.fromiter((len(p) for p in polylines), dtype=np.int64, count=len(polylines))
    off = np.zeros(len(polylines) + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    verts = np.concatenate([p.vertices if hasattr(p, "vertices") else np.asarray(p, float) for p in polylines])
    pairs = np.asarray(sorted(pair_items), dtype=np.int32).reshape(-1, 2)
    raw, lk, flags = _native.context().evaluate_pairs(verts, off, pairs, ds_mode((choice or KernelChoice()).ds_variant))
    _raise_for_flags(raw, flags)
    return {(int(i), int(j)): int(v) for (i, j), v in zip(pairs.tolist(), lk.tolist())}


def _prepare(model, choice, excluded, params, timings=None, packed=False):
    """PLS + discretization (certify.py:130-138); polylines copied back from the device."""
    params = params or DiscretizationParams()
    tick = time.perf_counter()
    ctx = upload(model)
    ctx.potential_link_search(excluded_keys(excluded))
    pair_list = PairList._from_sorted_array(ctx.get_pairs(), excluded)
    tock = time.perf_counter()
    try:
        ctx.discretize(model.xi, params.epsilon, params.max_passes, params.max_subsegments)
    except _native.DiscretizeFailure as fail:
        raise_for_failure(fail, params)
    verts, off = ctx.get_polylines()
    if timings is not None:
        timings["pls"] = tock - tick
        timings["discretize"] = time.perf_counter() - tock
    if packed:
        return pair_list, verts, off
    return pair_list, split_polylines(verts, off)


def _round_array(raw):
    """Python round() (half-to-even) per value plus the NaN / ambiguity flags (kernels.py:68-73)."""
    raw = np.asarray(raw, dtype=np.float64)
    nan = np.isnan(raw)
    r = np.rint(np.where(nan, 0.0, raw))
    flags = np.where(nan, _native.FLAG_NAN, 0).astype(np.uint8)
    flags[~nan & (np.abs(raw - r) > ROUNDING_THRESHOLD)] |= _native.FLAG_AMBIGUOUS
    return r.astype(np.int64), flags


def _bh_evaluate(model, choice, excluded, params, timings=None):
    """Barnes-Hut certificate values: PLS + discretization on the device, then
    every candidate pair through one batched moment-forest traversal."""
    pair_list, verts, off = _prepare(model, choice, excluded, params, timings, packed=True)
    pairs = pair_list.array.astype(np.int64).reshape(-1, 2)
    tick = time.perf_counter()
    raw, est, beta_used, reran = barneshut.evaluate_pairs_packed(verts, off, pairs, choice.bh)
    lk, flags = _round_array(raw)
    if timings is not None:
        timings["kernel"] = time.perf_counter() - tick
    # diagnostics of the reran pairs, keys in compute_link's order (kernels.py:60-67)
    diagnostics = {(int(pairs[k, 0]), int(pairs[k, 1])): {"e_estimate": float(est[k]),
                                                          "beta_used": float(beta_used[k]),
                                                          "reran": True, "raw": float(raw[k])}
                   for k in np.nonzero(reran)[0]}
    return pairs, raw, lk, flags, diagnostics


def compute_linking_matrix(
    model: CurveModel,
    choice: KernelChoice | None = None,
    excluded=(),
    threads: int = 1,
    params: DiscretizationParams | None = None,
    timings: dict | None = None,
) -> LinkMatrix:
    """Full pipeline: potential link search, discretization, kernel per pair (certify.py:141-166)."""
    choice = choice or KernelChoice()
    require_gpu_kernel(choice)
    if model.num_loops < 1:
        raise ValidationError("model has no loops")
    if choice.method == BARNES_HUT:
        pairs, raw, lk, flags, diagnostics = _bh_evaluate(model, choice, excluded, params, timings)
        _raise_for_flags(raw, flags)
        keep = lk != 0
        arr = np.concatenate([pairs[keep], lk[keep, None]], axis=1) if len(pairs) else np.zeros((0, 3), np.int64)
        return LinkMatrix._from_array(model.num_loops, arr, model_digest(model), choice.tag, diagnostics)
    if model.num_loops == 1:
        arr = np.zeros((0, 3), dtype=np.int64)
        if timings is not None:
            timings.update(pls=0.0, discretize=0.0, kernel=0.0)
        digest = model_digest(model)
    else:
        snap, digest_of = snapshot_and_digest(model, _dist())
        ctx = _native.context()
        try:
            with ctx.session:   # the result views stay ours until copied into arr
                pairs, raw, lk, flags, _ = run_device_pipeline(model, excluded, params, timings, ctx=ctx,
                                                               snapshot=snap, mode=ds_mode(choice.ds_variant))
                _raise_for_flags(raw, flags)
                keep = lk != 0
                arr = np.empty((int(keep.sum()), 3), dtype=np.int64)
                arr[:, :2] = pairs[keep]
                arr[:, 2] = lk[keep]
        except Exception:
            digest_of()           # a serialization error would have surfaced last in the reference
            raise
        digest = digest_of()
    return LinkMatrix._from_array(model.num_loops, arr, digest, choice.tag, {})


def verify(
    model: CurveModel,
    reference: LinkMatrix,
    choice: KernelChoice | None = None,
    early_exit: bool = False,
    excluded=(),
    threads: int = 1,
    params: DiscretizationParams | None = None,
) -> VerificationReport:
    """Recompute pairwise links and diff against a reference certificate (certify.py:169-221)."""
    choice = choice or KernelChoice()
    require_gpu_kernel(choice)
    if model.num_loops != reference.num_loops:
        return VerificationReport(
            FAIL,
            message=(f"loop count mismatch: model has {model.num_loops}, "
                     f"certificate has {reference.num_loops}"),
        )
    if choice.method == BARNES_HUT:
        _warn_digest(model_digest(model), reference)
        if model.num_loops < 1:
            raise ValidationError("model has no loops")
        pairs, raw, lk, flags, _ = _bh_evaluate(model, choice, excluded, params)
        return diff_arrays(reference.array, pairs, raw, lk, flags, early_exit)
    # the digest (host, native) overlaps the device pipeline; its check and
    # warning come first, as in the reference (certify.py:188-193)
    snap, digest_of = snapshot_and_digest(model, _dist())
    ctx = None
    try:
        if model.num_loops < 1:
            raise ValidationError("model has no loops")
        if model.num_loops == 1:
            pairs = np.zeros((0, 2), dtype=np.int32)
            raw = np.zeros(0)
            lk = np.zeros(0, dtype=np.int64)
            flags = np.zeros(0, dtype=np.uint8)
        else:
            ctx = _native.context()
            ctx.session.acquire()   # the result views stay ours through the diff
            try:
                if early_exit:   # single GPU: pairs past the first failure are cancelled on the device
                    arr = reference.array
                    ctx.set_early_exit(_pair_keys(arr[:, :2]).astype(np.uint64), arr[:, 2])
                try:
                    pairs, raw, lk, flags, _ = run_device_pipeline(model, excluded, params, ctx=ctx, snapshot=snap,
                                                                   mode=ds_mode(choice.ds_variant))
                finally:
                    if early_exit:
                        ctx.set_early_exit(None)
            except Exception:
                ctx.session.release()
                raise
    except Exception:
        _warn_digest(digest_of(), reference)
        raise
    # the diff runs while the digest finishes; its outcome (report or error) is
    # delivered after the digest warning, the reference's order
    try:
        report, err = diff_arrays(reference.array, pairs, raw, lk, flags, early_exit), None
    except Exception as exc:  # noqa: BLE001 - re-raised below, after the warning
        report, err = None, exc
    finally:
        if ctx is not None:
            ctx.session.release()
    _warn_digest(digest_of(), reference)
    if err is not None:
        raise err
    return report


def _warn_digest(digest, reference):
    if reference.model_digest and digest != reference.model_digest:
        warnings.warn("model digest differs from certificate digest (deformed model?)", stacklevel=3)


def _lookup(sorted_keys, query):
    """Index of each query key in sorted_keys, -1 where absent."""
    if not len(sorted_keys):
        return np.full(len(query), -1, dtype=np.int64)
    pos = np.minimum(np.searchsorted(sorted_keys, query), len(sorted_keys) - 1)
    return np.where(sorted_keys[pos] == query, pos, -1)


def diff_arrays(ref_arr, pairs, raw, lk, flags, early_exit=False):
    """Vectorized verify diff (certify.py:194-221) over sorted reference entries
    and the device results of the sorted candidate pairs."""
    ref_arr = np.asarray(ref_arr, dtype=np.int64).reshape(-1, 3)
    ref_keys = _pair_keys(ref_arr[:, :2])
    ref_vals = ref_arr[:, 2]
    cand_keys = _pair_keys(pairs)
    lk = np.asarray(lk, dtype=np.int64)
    # ordering = sorted(ref) + sorted(candidate - ref)   (certify.py:196-198)
    ref_cidx = _lookup(cand_keys, ref_keys)                         # -1: not a candidate -> 0
    extra_idx = np.nonzero(_lookup(ref_keys, cand_keys) < 0)[0]
    order_keys = np.concatenate([ref_keys, cand_keys[extra_idx]])
    order_cidx = np.concatenate([ref_cidx, extra_idx])
    order_want = np.concatenate([ref_vals, np.zeros(len(extra_idx), dtype=np.int64)])
    order_got = np.where(order_cidx >= 0, lk[np.maximum(order_cidx, 0)] if len(lk) else 0, 0)
    mism = order_got != order_want
    if early_exit:
        hit = np.nonzero(mism)[0]
        stop = int(hit[0]) if len(hit) else len(order_keys) - 1
        evaluated = order_cidx[: stop + 1]
        evaluated = evaluated[evaluated >= 0]
        _raise_for_flags(raw, flags, evaluated)
        if not len(hit):
            return VerificationReport(PASS)
        f = int(hit[0])
        pair = (int(order_keys[f] >> 32), int(order_keys[f] & 0xFFFFFFFF))
        report = _classify([pair], [int(order_want[f])], [int(order_got[f])])
        report.status = ABORTED
        report.first_failure = pair
        return report
    computed_order = order_cidx[order_cidx >= 0]
    _raise_for_flags(raw, flags, computed_order)
    idx = np.nonzero(mism)[0]
    idx = idx[np.argsort(order_keys[idx], kind="stable")]
    bad_pairs = [(int(k >> 32), int(k & 0xFFFFFFFF)) for k in order_keys[idx].tolist()]
    return _classify(bad_pairs, order_want[idx].tolist(), order_got[idx].tolist())


def _classify(pairs, want, got):
    destroyed, created, changed = [], [], []
    for pair, w, g in zip(pairs, want, got):
        if w != 0 and g == 0:
            destroyed.append(pair)
        elif w == 0 and g != 0:
            created.append(pair)
        else:
            changed.append(pair)
    status = PASS if not (destroyed or created or changed) else FAIL
    return VerificationReport(status, destroyed, created, changed)


def diff_matrices(a: LinkMatrix, b: LinkMatrix) -> VerificationReport:
    """Diff two certificates, treating `a` as the reference (certify.py:224-231)."""
    if a.num_loops != b.num_loops:
        return VerificationReport(FAIL, message=f"loop count mismatch: {a.num_loops} vs {b.num_loops}")
    return _diff(a.as_dict(), b.as_dict())


def _diff(ref, computed):
    """certify.py:234-250."""
    keys = sorted(set(ref) | set(computed))
    want = [ref.get(p, 0) for p in keys]
    got = [computed.get(p, 0) for p in keys]
    sel = [k for k in range(len(keys)) if want[k] != got[k]]
    return _classify([keys[k] for k in sel], [want[k] for k in sel], [got[k] for k in sel])
