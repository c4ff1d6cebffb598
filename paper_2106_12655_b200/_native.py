"""ctypes binding of liblinkcert_b200.so (include/linkcert_b200.h).

There is no CPU fallback: if the library or a CUDA device is missing, every
entry point raises NativeUnavailable.  The library is built in-tree by
``python -m paper_2106_12655_b200.build`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "liblinkcert_b200.so"

LC_OK = 0
LC_ERR_CUDA = 1
LC_ERR_ARG = 2
LC_ERR_STATE = 3
LC_ERR_DISCRETIZE = 4
LC_ERR_VALIDATION = 5

GAUSS_PHASE = 0
GAUSS_ATAN = 1
GAUSS_REF = 2
GAUSS_ANGLESUM = 3
GAUSS_MODES = {"phase": GAUSS_PHASE, "atan": GAUSS_ATAN, "ref": GAUSS_REF}   # arithmetic forms of the "atan" variant

FLAG_NAN = 1
FLAG_AMBIGUOUS = 2

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_int64_p = ctypes.POINTER(ctypes.c_int64)
_c_int32_p = ctypes.POINTER(ctypes.c_int32)
_c_uint8_p = ctypes.POINTER(ctypes.c_uint8)
_c_float_p = ctypes.POINTER(ctypes.c_float)
_vp = ctypes.c_void_p

# name -> (restype, argtypes); exactly the symbols of include/linkcert_b200.h
SIGNATURES = {
    "lc_abi_version": (ctypes.c_int, []),
    "lc_last_error": (ctypes.c_char_p, []),
    "lc_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "lc_create": (_vp, [ctypes.c_int]),
    "lc_destroy": (None, [_vp]),
    "lc_set_stream": (ctypes.c_int, [_vp, _vp]),
    "lc_synchronize": (ctypes.c_int, [_vp]),
    "lc_evaluate_pairs": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64,
                                          ctypes.c_int, _vp, _vp, _vp]),
    "lc_link_direct": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int, _vp]),
    "lc_segment_pair_lambda": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp]),
    "lc_last_gauss_ms": (ctypes.c_int, [_vp, _c_float_p]),
    "lc_stage_polylines": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int,
                                           _c_int64_p]),
    "lc_gauss_run": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _vp]),
    "lc_gauss_reduce": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "lc_gauss_run_pairs": (ctypes.c_int, [_vp, ctypes.c_int]),
    "lc_gauss_event_ms": (ctypes.c_int, [_vp, _c_float_p]),
    "lc_probe_fp64_peak": (ctypes.c_int, [_vp, _c_double_p, _c_float_p]),
    "lc_probe_fp64_dmma_peak": (ctypes.c_int, [_vp, _c_double_p, _c_float_p]),
    "lc_model_upload": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int64]),
    "lc_model_upload_polylines": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64]),
    "lc_model_upload_polyline_ptrs": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64]),
    "lc_model_digest_polylines": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p]),
    "lc_model_digest_polylines_stream": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int,
                                                        ctypes.c_char_p]),
    "lc_tight_boxes": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, _vp, _vp]),
    "lc_loop_boxes": (ctypes.c_int, [_vp, _vp, _vp]),
    "lc_potential_link_search": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _c_int64_p]),
    "lc_get_pairs": (ctypes.c_int, [_vp, _vp]),
    "lc_set_pairs": (ctypes.c_int, [_vp, _vp, ctypes.c_int64]),
    "lc_discretize": (ctypes.c_int, [_vp, ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int64,
                                      _c_int64_p, ctypes.POINTER(ctypes.c_int)]),
    "lc_discretize_error": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                            _vp, ctypes.c_int64, _c_int64_p]),
    "lc_get_polylines": (ctypes.c_int, [_vp, _vp, _vp]),
    "lc_prepare_gauss": (ctypes.c_int, [_vp, ctypes.c_int, _c_int64_p]),
    "lc_evaluate_staged": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _vp, _vp]),
    "lc_run_pipeline": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                        ctypes.c_int64, ctypes.c_int, _c_int64_p]),
    "lc_get_results": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "lc_result_views": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                        ctypes.POINTER(_vp), _c_int64_p]),
    "lc_stage_times": (ctypes.c_int, [_vp, _c_float_p]),
    "lc_set_stage_detail": (ctypes.c_int, [_vp, ctypes.c_int]),
    "lc_model_json_bound": (ctypes.c_int64, [_vp, ctypes.c_int64]),
    "lc_model_json": (ctypes.c_int64, [_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, _vp, ctypes.c_int64]),
    "lc_float_repr": (ctypes.c_int, [ctypes.c_double, ctypes.c_char_p]),
    "lc_last_run_fused": (ctypes.c_int, [_vp]),
    "lc_host_alloc": (_vp, [ctypes.c_int64]),
    "lc_host_free": (None, [_vp]),
    "lc_run_pipeline_shard_async": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                                   ctypes.c_int, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_int64)]),
    "lc_shard_finish": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int)]),
    "lc_nccl_version": (ctypes.c_int, []),
    "lc_comm_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "lc_comm_init": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int, ctypes.c_int]),
    "lc_comm_destroy": (ctypes.c_int, [_vp]),
    "lc_run_pipeline_sharded": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                                ctypes.c_int, ctypes.c_int64, ctypes.c_int, _c_int64_p]),
    "lc_shard_bounds": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
    "lc_set_early_exit": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int]),
    "lc_early_exit_stats": (ctypes.c_int, [_vp, _c_int64_p, _c_int64_p]),
    "lc_get_stream": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    "lc_float_repr_many": (ctypes.c_int64, [_vp, ctypes.c_int64, ctypes.c_int, _vp, ctypes.c_int64]),
    "lc_model_digest": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p]),
    "lc_sha256_hex": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int, ctypes.c_char_p]),
    "lc_launch_count": (ctypes.c_longlong, []),
    "lc_bh_forest_build": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int64, ctypes.POINTER(_vp)]),
    "lc_bh_forest_free": (ctypes.c_int, [_vp, _vp]),
    "lc_bh_forest_sizes": (ctypes.c_int, [_vp, _c_int64_p, _c_int64_p, _c_int64_p, ctypes.POINTER(ctypes.c_int)]),
    "lc_bh_forest_nodes": (ctypes.c_int, [_vp] * 18),
    "lc_bh_far_field": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int, _c_double_p]),
    "lc_bh_eval": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int64, _vp, ctypes.c_int, ctypes.c_double, _vp, _vp,
                                   _c_int64_p]),
}


def launch_count():
    return int(load_library().lc_launch_count())


def model_digest(coeffs, t, loop_off, closed=None, nthreads=0):
    """SHA-256 hex of the canonical model JSON (host C++; GIL released); None if non-finite."""
    lib = load_library()
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    loop_off = np.ascontiguousarray(loop_off, dtype=np.int64)
    cl = None if closed is None else np.ascontiguousarray(closed, dtype=np.uint8)
    out = ctypes.create_string_buffer(65)
    rc = lib.lc_model_digest(_ptr(coeffs), _ptr(t), _ptr(loop_off), _ptr(cl), len(loop_off) - 1, int(nthreads), out)
    return None if rc != 0 else out.value.decode()


def model_digest_polylines(vptrs, loop_off, nthreads=0):
    """model_digest of closed from_polyline loops given by their vertex-array
    addresses (vptrs uint64 (L)); None if a coordinate is non-finite."""
    lib = load_library()
    vptrs = np.ascontiguousarray(vptrs, dtype=np.uint64)
    loop_off = np.ascontiguousarray(loop_off, dtype=np.int64)
    out = ctypes.create_string_buffer(65)
    rc = lib.lc_model_digest_polylines(_ptr(vptrs), _ptr(loop_off), len(loop_off) - 1, int(nthreads), out)
    if rc == -2:
        raise NativeError(LC_ERR_ARG, "lc_model_digest_polylines: null loop pointer")
    return None if rc != 0 else out.value.decode()


def model_digest_polylines_stream(vptrs, loop_off, ready, nthreads=0):
    """model_digest_polylines while vptrs (uint64 (L)) / loop_off (int64 (L+1)) are
    being filled in loop order; ready (int64 (1)) holds the count of filled loops
    (negative: abort).  Returns the digest, None for a non-finite coordinate, or
    raises Aborted."""
    lib = load_library()
    assert vptrs.dtype == np.uint64 and loop_off.dtype == np.int64 and ready.dtype == np.int64
    out = ctypes.create_string_buffer(65)
    rc = lib.lc_model_digest_polylines_stream(_ptr(vptrs), _ptr(loop_off), len(loop_off) - 1, _ptr(ready),
                                              int(nthreads), out)
    if rc == -2:
        raise NativeError(LC_ERR_ARG, "lc_model_digest_polylines_stream: null loop pointer")
    if rc == -3:
        raise DigestAborted()
    return None if rc != 0 else out.value.decode()


class DigestAborted(Exception):
    """A streamed digest whose input was withdrawn (the model is not all closed polylines)."""


def comm_unique_id():
    """128-byte NCCL unique id for a new library communicator (call on rank 0)."""
    out = ctypes.create_string_buffer(128)
    rc = load_library().lc_comm_unique_id(out)
    if rc != LC_OK:
        raise NativeError(rc, load_library().lc_last_error().decode(errors="replace"))
    return out.raw


def nccl_version():
    return int(load_library().lc_nccl_version())


def sha256_hex(data, force_portable=False):
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    out = ctypes.create_string_buffer(65)
    has = load_library().lc_sha256_hex(_ptr(buf), buf.size, int(force_portable), out)
    return out.value.decode(), bool(has)


def model_json(coeffs, t, loop_off, closed=None, nthreads=0):
    """Canonical json-curves bytes of a packed model (host C++, GIL released)."""
    lib = load_library()
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    loop_off = np.ascontiguousarray(loop_off, dtype=np.int64)
    L = len(loop_off) - 1
    cl = None if closed is None else np.ascontiguousarray(closed, dtype=np.uint8)
    cap = lib.lc_model_json_bound(_ptr(loop_off), L)
    buf = np.empty(cap, dtype=np.uint8)
    n = lib.lc_model_json(_ptr(coeffs), _ptr(t), _ptr(loop_off), _ptr(cl), L, int(nthreads),
                          buf.ctypes.data_as(ctypes.c_void_p), cap)
    if n == -1:
        return None
    if n < 0:
        raise NativeError(LC_ERR_STATE, "lc_model_json: buffer too small")
    return memoryview(buf)[:n]


_pinned_ok = None


def pinned_empty(shape, dtype=np.float64):
    """numpy array in page-locked host memory (freed with the array); plain numpy
    memory when no device is usable (the arrays are storage, not a compute path)."""
    global _pinned_ok
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) * dtype.itemsize
    if n > 0 and _pinned_ok is not False:
        try:
            lib = load_library()
            ptr = lib.lc_host_alloc(n)
        except NativeUnavailable:
            ptr = None
        _pinned_ok = bool(ptr)
        if ptr:
            raw = (ctypes.c_char * n).from_address(ptr)
            import weakref

            weakref.finalize(raw, lib.lc_host_free, ptr)
            return np.frombuffer(raw, dtype=dtype).reshape(shape)
    return np.empty(shape, dtype=dtype)


def pinned_copy(a):
    out = pinned_empty(a.shape, a.dtype)
    np.copyto(out, a)
    return out


def float_repr(x):
    out = ctypes.create_string_buffer(40)
    n = load_library().lc_float_repr(float(x), out)
    return out.raw[:n].decode()


def float_repr_many(xs, use_tochars=False):
    """repr of every double in xs (test hook for the digest formatter)."""
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    buf = np.empty(26 * len(xs) + 1, dtype=np.uint8)
    n = load_library().lc_float_repr_many(_ptr(xs), len(xs), int(bool(use_tochars)), _ptr(buf), len(buf))
    return buf[:n].tobytes().decode().split("\n")[:-1]

# lc_discretize_error kinds
DISC_OK = 0
DISC_ZERO_LENGTH = 1
DISC_CURVES_INTERSECT = 2
DISC_SUBSEG_BUDGET = 3
DISC_PASS_BUDGET = 4
DISC_INVALID_POLYLINE = 5


class DiscretizeFailure(Exception):
    """Structured discretization failure reported by the device (mapped to the
    reference exception types by paper_2106_12655_b200.discretize)."""

    def __init__(self, kind, detail, loops):
        super().__init__(f"discretization failure kind={kind} detail={detail} loops={loops}")
        self.kind = kind
        self.detail = detail
        self.loops = tuple(int(x) for x in loops)


class NativeUnavailable(RuntimeError):
    """The sm_100a library or a CUDA device is not available (no CPU fallback)."""


class NativeError(RuntimeError):
    def __init__(self, code, message):
        super().__init__(f"liblinkcert_b200 error {code}: {message}")
        self.code = code


_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load and type the shared library (no device needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        path = Path(os.environ.get("LINKCERT_LIB", LIB_PATH))   # A/B builds (tools/); default in-tree
        if not path.exists():
            raise NativeUnavailable(
                f"{path} is missing; build it with `python -m paper_2106_12655_b200.build`"
            )
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def _check(rc):
    if rc != LC_OK:
        msg = _lib.lc_last_error().decode(errors="replace")
        raise NativeError(rc, msg)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


def default_device():
    for key in ("LINKCERT_DEVICE", "LOCAL_RANK"):
        if key in os.environ:
            return int(os.environ[key])
    return 0


class Context:
    """One library context (device + stream + cached device buffers)."""

    def __init__(self, device=None):
        lib = load_library()
        n = ctypes.c_int(0)
        if lib.lc_device_count(ctypes.byref(n)) != LC_OK or n.value == 0:
            raise NativeUnavailable("no CUDA device visible to liblinkcert_b200 (there is no CPU fallback)")
        self.device = default_device() if device is None else device
        if self.device >= n.value:
            self.device = self.device % n.value
        h = lib.lc_create(self.device)
        if not h:
            raise NativeUnavailable(f"lc_create({self.device}) failed: {lib.lc_last_error().decode()}")
        self.handle = ctypes.c_void_p(h)
        self.lib = lib
        # one re-entrant lock: every call takes it, and a caller holds it (as `session`)
        # across upload -> pipeline -> use of the result views, so concurrent callers on
        # this context can neither interleave models nor overwrite each other's views
        self.lock = threading.RLock()
        self.session = self.lock

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and self.lib is not None:
            try:
                self.lib.lc_destroy(h)
            except Exception:
                pass

    # ---- Gauss sum ----------------------------------------------------------
    def evaluate_pairs(self, verts, vert_off, pairs, mode=GAUSS_PHASE):
        """raw, lk, flags for every pair (host arrays in, host arrays out)."""
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        vert_off = np.ascontiguousarray(vert_off, dtype=np.int64)
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        P = pairs.shape[0]
        raw = np.empty(P, dtype=np.float64)
        lk = np.empty(P, dtype=np.int64)
        flags = np.empty(P, dtype=np.uint8)
        with self.lock:
            _check(self.lib.lc_evaluate_pairs(self.handle, _ptr(verts), _ptr(vert_off), len(vert_off) - 1,
                                              _ptr(pairs), P, int(mode), _ptr(raw), _ptr(lk), _ptr(flags)))
        return raw, lk, flags

    def link_direct(self, loop1, loop2, mode=GAUSS_PHASE):
        a = np.ascontiguousarray(loop1, dtype=np.float64)
        b = np.ascontiguousarray(loop2, dtype=np.float64)
        out = ctypes.c_double(0.0)
        with self.lock:
            _check(self.lib.lc_link_direct(self.handle, _ptr(a), a.shape[0], _ptr(b), b.shape[0], int(mode),
                                           ctypes.byref(out)))
        return out.value

    def segment_pair_lambda(self, quads):
        q = np.ascontiguousarray(quads, dtype=np.float64).reshape(-1, 12)
        out = np.empty(q.shape[0], dtype=np.float64)
        with self.lock:
            _check(self.lib.lc_segment_pair_lambda(self.handle, _ptr(q), q.shape[0], _ptr(out)))
        return out

    def last_gauss_ms(self):
        ms = ctypes.c_float(0.0)
        _check(self.lib.lc_last_gauss_ms(self.handle, ctypes.byref(ms)))
        return ms.value

    def stage_polylines(self, verts, vert_off, pairs, mode=GAUSS_PHASE):
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        vert_off = np.ascontiguousarray(vert_off, dtype=np.int64)
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        n = ctypes.c_int64(0)
        with self.lock:
            _check(self.lib.lc_stage_polylines(self.handle, _ptr(verts), _ptr(vert_off), len(vert_off) - 1,
                                               _ptr(pairs), pairs.shape[0], int(mode), ctypes.byref(n)))
        self._staged_pairs = pairs.shape[0]
        return n.value

    def gauss_run(self, mode, item_begin, item_end, partials_dev_ptr=None):
        with self.lock:
            _check(self.lib.lc_gauss_run(self.handle, int(mode), int(item_begin), int(item_end),
                                         ctypes.c_void_p(partials_dev_ptr) if partials_dev_ptr else None))

    def gauss_run_pairs(self, mode):
        """Pair-claiming kernel over the staged pairs (timing A/B; gauss_event_ms reads it)."""
        with self.lock:
            _check(self.lib.lc_gauss_run_pairs(self.handle, int(mode)))

    def gauss_reduce(self, partials_dev_ptr=None):
        P = self._staged_pairs
        raw = np.empty(P, dtype=np.float64)
        lk = np.empty(P, dtype=np.int64)
        flags = np.empty(P, dtype=np.uint8)
        with self.lock:
            _check(self.lib.lc_gauss_reduce(self.handle,
                                            ctypes.c_void_p(partials_dev_ptr) if partials_dev_ptr else None,
                                            _ptr(raw), _ptr(lk), _ptr(flags)))
        return raw, lk, flags

    def gauss_event_ms(self):
        ms = ctypes.c_float(0.0)
        _check(self.lib.lc_gauss_event_ms(self.handle, ctypes.byref(ms)))
        return ms.value

    def synchronize(self):
        _check(self.lib.lc_synchronize(self.handle))

    def set_stream(self, cuda_stream_ptr):
        """Launch on a caller stream (e.g. torch.cuda.current_stream().cuda_stream); 0/None = own stream."""
        with self.lock:
            _check(self.lib.lc_set_stream(self.handle, ctypes.c_void_p(cuda_stream_ptr) if cuda_stream_ptr else None))

    # ---- model pipeline -------------------------------------------------------
    def tight_boxes(self, coeffs, t):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(-1, 4, 3)
        t = np.ascontiguousarray(t, dtype=np.float64).reshape(-1, 2)
        m = coeffs.shape[0]
        lo = np.empty((m, 3))
        hi = np.empty((m, 3))
        with self.lock:
            _check(self.lib.lc_tight_boxes(self.handle, _ptr(coeffs), _ptr(t), m, _ptr(lo), _ptr(hi)))
        return lo, hi

    def upload_model(self, coeffs, t, loop_off):
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        loop_off = np.ascontiguousarray(loop_off, dtype=np.int64)
        with self.lock:
            _check(self.lib.lc_model_upload(self.handle, _ptr(coeffs), _ptr(t), _ptr(loop_off), len(loop_off) - 1))
        self._L = len(loop_off) - 1

    def upload_model_polylines(self, verts, loop_off):
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        loop_off = np.ascontiguousarray(loop_off, dtype=np.int64)
        with self.lock:
            _check(self.lib.lc_model_upload_polylines(self.handle, _ptr(verts), _ptr(loop_off), len(loop_off) - 1))
        self._L = len(loop_off) - 1

    def upload_model_polyline_ptrs(self, vptrs, loop_off):
        """Closed polylines from one vertex array per loop (addresses in vptrs); the
        library gathers them into its pinned staging buffer, the copy runs async."""
        vptrs = np.ascontiguousarray(vptrs, dtype=np.uint64)
        loop_off = np.ascontiguousarray(loop_off, dtype=np.int64)
        with self.lock:
            _check(self.lib.lc_model_upload_polyline_ptrs(self.handle, _ptr(vptrs), _ptr(loop_off),
                                                          len(loop_off) - 1))
        self._L = len(loop_off) - 1

    def loop_boxes(self):
        lo = np.empty((self._L, 3))
        hi = np.empty((self._L, 3))
        with self.lock:
            _check(self.lib.lc_loop_boxes(self.handle, _ptr(lo), _ptr(hi)))
        return lo, hi

    def potential_link_search(self, excluded_keys=None):
        ex = np.ascontiguousarray(excluded_keys if excluded_keys is not None else [], dtype=np.uint64)
        n = ctypes.c_int64(0)
        with self.lock:
            _check(self.lib.lc_potential_link_search(self.handle, _ptr(ex), ex.size, ctypes.byref(n)))
        self._staged_pairs = n.value
        return n.value

    def get_pairs(self):
        out = np.empty((self._staged_pairs, 2), dtype=np.int32)
        with self.lock:
            _check(self.lib.lc_get_pairs(self.handle, _ptr(out)))
        return out

    def set_pairs(self, pairs):
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        with self.lock:
            _check(self.lib.lc_set_pairs(self.handle, _ptr(pairs), pairs.shape[0]))
        self._staged_pairs = pairs.shape[0]

    def _disc_error(self):
        kind = ctypes.c_int(0)
        detail = ctypes.c_int(0)
        n = ctypes.c_int64(0)
        _check(self.lib.lc_discretize_error(self.handle, ctypes.byref(kind), ctypes.byref(detail), None, 0,
                                            ctypes.byref(n)))
        loops = np.zeros(max(n.value, 1), dtype=np.int64)
        _check(self.lib.lc_discretize_error(self.handle, ctypes.byref(kind), ctypes.byref(detail), _ptr(loops),
                                            n.value, ctypes.byref(n)))
        return DiscretizeFailure(kind.value, detail.value, loops[:n.value].tolist())

    def discretize(self, xi, epsilon, max_passes, max_subsegments):
        """Run device discretization; returns (n_vertices, passes) or raises DiscretizeFailure."""
        nv = ctypes.c_int64(0)
        passes = ctypes.c_int(0)
        with self.lock:
            rc = self.lib.lc_discretize(self.handle, float(xi), float(epsilon), int(max_passes), int(max_subsegments),
                                        ctypes.byref(nv), ctypes.byref(passes))
            if rc in (LC_ERR_DISCRETIZE, LC_ERR_VALIDATION):
                raise self._disc_error()
            _check(rc)
        self._nverts = nv.value
        return nv.value, passes.value

    def get_polylines(self):
        off = np.empty(self._L + 1, dtype=np.int64)
        with self.lock:
            _check(self.lib.lc_get_polylines(self.handle, None, _ptr(off)))
            verts = np.empty((int(off[-1]) if len(off) else 0, 3))
            _check(self.lib.lc_get_polylines(self.handle, _ptr(verts), None))
        return verts, off

    def evaluate_staged(self, mode=GAUSS_PHASE):
        P = self._staged_pairs
        raw = np.empty(P)
        lk = np.empty(P, dtype=np.int64)
        flags = np.empty(P, dtype=np.uint8)
        with self.lock:
            _check(self.lib.lc_evaluate_staged(self.handle, int(mode), _ptr(raw), _ptr(lk), _ptr(flags)))
        return raw, lk, flags

    def prepare_gauss(self, mode=GAUSS_PHASE):
        n = ctypes.c_int64(0)
        with self.lock:
            _check(self.lib.lc_prepare_gauss(self.handle, int(mode), ctypes.byref(n)))
        return n.value

    def run_pipeline(self, excluded_keys, xi, epsilon, max_passes, max_subsegments, mode=GAUSS_PHASE):
        """PLS -> discretize -> Gauss on the uploaded model; returns P (results stay on device)."""
        ex = np.ascontiguousarray(excluded_keys if excluded_keys is not None else [], dtype=np.uint64)
        n = ctypes.c_int64(0)
        with self.lock:
            rc = self.lib.lc_run_pipeline(self.handle, _ptr(ex), ex.size, float(xi), float(epsilon), int(max_passes),
                                          int(max_subsegments), int(mode), ctypes.byref(n))
            if rc in (LC_ERR_DISCRETIZE, LC_ERR_VALIDATION):
                raise self._disc_error()
            _check(rc)
        self._staged_pairs = n.value
        return n.value

    def get_results(self):
        P = self._staged_pairs
        raw = np.empty(P)
        lk = np.empty(P, dtype=np.int64)
        flags = np.empty(P, dtype=np.uint8)
        with self.lock:
            _check(self.lib.lc_get_results(self.handle, _ptr(raw), _ptr(lk), _ptr(flags)))
        return raw, lk, flags

    def run_pipeline_shard_async(self, excluded_keys, xi, epsilon, max_passes, max_subsegments, mode, shard,
                                 shards):
        """Enqueue the fused run of item shard `shard` of `shards` (>= 2) without a
        host sync; returns (device pointer of the partials, entries) or None when
        the staged path must run.  Complete with shard_finish()."""
        ex = np.ascontiguousarray(excluded_keys if excluded_keys is not None else [], dtype=np.uint64)
        ptr, cap = _vp(), ctypes.c_int64(0)
        with self.lock:
            _check(self.lib.lc_run_pipeline_shard_async(self.handle, _ptr(ex), ex.size, float(xi), float(epsilon),
                                                        int(max_passes), int(max_subsegments), int(mode),
                                                        int(shard), int(shards), ctypes.byref(ptr),
                                                        ctypes.byref(cap)))
        return None if cap.value <= 0 else (ptr.value, cap.value)

    def shard_finish(self):
        """Reduce + export + the one host sync of an async sharded run; True: results ready."""
        fused = ctypes.c_int(0)
        with self.lock:
            rc = self.lib.lc_shard_finish(self.handle, ctypes.byref(fused))
            if rc in (LC_ERR_DISCRETIZE, LC_ERR_VALIDATION):
                raise self._disc_error()
            _check(rc)
        return bool(fused.value)

    # ---- multi-GPU (library-owned NCCL communicator) ------------------------
    def comm_init(self, unique_id, world, rank):
        """Join the communicator `unique_id` (128 bytes from comm_unique_id() on rank 0)."""
        with self.lock:
            _check(self.lib.lc_comm_init(self.handle, bytes(unique_id), int(world), int(rank)))
        self.comm = (int(world), int(rank))

    def comm_destroy(self):
        with self.lock:
            _check(self.lib.lc_comm_destroy(self.handle))
        self.comm = None

    def run_pipeline_sharded(self, excluded_keys, xi, epsilon, max_passes, max_subsegments, mode=GAUSS_PHASE):
        """run_pipeline over the communicator: this rank's cost-balanced share of the
        Gauss sum, partials exchanged in the library; full results on every rank."""
        ex = np.ascontiguousarray(excluded_keys if excluded_keys is not None else [], dtype=np.uint64)
        n = ctypes.c_int64(0)
        with self.lock:
            rc = self.lib.lc_run_pipeline_sharded(self.handle, _ptr(ex), ex.size, float(xi), float(epsilon),
                                                  int(max_passes), int(max_subsegments), int(mode), ctypes.byref(n))
            if rc in (LC_ERR_DISCRETIZE, LC_ERR_VALIDATION):
                raise self._disc_error()
            _check(rc)
        self._staged_pairs = n.value
        return n.value

    def shard_bounds(self, shards):
        """Cost-balanced item ranges of the current work items: bounds (shards + 1)."""
        out = np.zeros(int(shards) + 1, dtype=np.int64)
        with self.lock:
            _check(self.lib.lc_shard_bounds(self.handle, int(shards), _ptr(out)))
        return out

    def set_early_exit(self, ref_keys=None, ref_lk=None):
        """Arm (certificate keys / values) or disarm (None) the device early exit."""
        if ref_keys is None:
            with self.lock:
                _check(self.lib.lc_set_early_exit(self.handle, None, None, 0, 0))
            return
        k = np.ascontiguousarray(ref_keys, dtype=np.uint64)
        v = np.ascontiguousarray(ref_lk, dtype=np.int64)
        with self.lock:
            _check(self.lib.lc_set_early_exit(self.handle, _ptr(k), _ptr(v), k.size, 1))

    def early_exit_stats(self):
        """(place of the first failing pair or -1, pairs evaluated or -1) of the last fused run."""
        f, n = ctypes.c_int64(0), ctypes.c_int64(0)
        with self.lock:
            _check(self.lib.lc_early_exit_stats(self.handle, ctypes.byref(f), ctypes.byref(n)))
        return f.value, n.value

    def stream_ptr(self):
        out = _vp()
        _check(self.lib.lc_get_stream(self.handle, ctypes.byref(out)))
        return out.value or 0

    def last_run_fused(self):
        """Path of the last run_pipeline: 0 staged, 1 fused, 2 fused graph replay."""
        with self.lock:
            return int(self.lib.lc_last_run_fused(self.handle))

    def result_views(self):
        """(pairs (P,2) int32, raw, lk, flags) views into the library's pinned result
        buffer — valid until the next pipeline call; copy what must be kept."""
        with self.lock:   # the output slots are per context, filled and read under its lock
            out = self.__dict__.get("_rv_out")
            if out is None:
                ptrs, n = [_vp() for _ in range(4)], ctypes.c_int64(0)
                out = self._rv_out = (ptrs, n, [ctypes.byref(p) for p in ptrs] + [ctypes.byref(n)])
            ptrs, n, refs = out
            _check(self.lib.lc_result_views(self.handle, *refs))
            P = n.value
            key = (P, ptrs[0].value, ptrs[1].value, ptrs[2].value, ptrs[3].value)
        if P == 0:
            return (np.zeros((0, 2), np.int32), np.zeros(0), np.zeros(0, np.int64), np.zeros(0, np.uint8))
        cached = getattr(self, "_views", None)
        if cached is not None and cached[0] == key:   # same buffer, same P: the same views
            return cached[1]

        def view(addr, ctype, shape):
            return np.ctypeslib.as_array(ctypes.cast(_vp(addr), ctypes.POINTER(ctype)), shape=shape)

        views = (view(key[1], ctypes.c_int32, (P, 2)), view(key[2], ctypes.c_double, (P,)),
                 view(key[3], ctypes.c_int64, (P,)), view(key[4], ctypes.c_uint8, (P,)))
        self._views = (key, views)
        return views

    def stage_times(self):
        """Device ms of the last pipeline's stages; None for a stage the last fused run
        did not time (stage detail off: only the Gauss stage)."""
        ms = (ctypes.c_float * 5)()
        with self.lock:
            _check(self.lib.lc_stage_times(self.handle, ms))
        names = ("pls", "discretize", "gauss", "reduce", "begin_to_reduce")
        return {k: (v if v >= 0.0 else None) for k, v in zip(names, ms)}

    def set_stage_detail(self, on):
        """Fused runs time every stage (on) or only the Gauss stage (off, the default)."""
        on = bool(on)
        if getattr(self, "_stage_detail", False) != on:
            with self.lock:
                _check(self.lib.lc_set_stage_detail(self.handle, int(on)))
            self._stage_detail = on

    def bh_forest(self, verts, loop_off):
        """Moment trees of closed polylines on this device (Barnes-Hut)."""
        return MomentForest(self, verts, loop_off)

    def probe_fp64_peak(self, dmma=False):
        """FP64 FLOP/s of the DFMA-chain probe (dmma=True: the FP64 tensor-core probe)."""
        flops = ctypes.c_double(0.0)
        ms = ctypes.c_float(0.0)
        fn = self.lib.lc_probe_fp64_dmma_peak if dmma else self.lib.lc_probe_fp64_peak
        with self.lock:
            _check(fn(self.handle, ctypes.byref(flops), ctypes.byref(ms)))
        return flops.value, ms.value


class MomentForest:
    """Device-resident moment trees of L closed polylines (lc_bh_forest_*):
    the Barnes-Hut trees of linkcert/barneshut.py:295-323, built on the GPU."""

    FIELDS = ("node_off", "left", "right", "start", "end", "prim_order", "node_lo", "node_hi", "center", "radius",
              "cm", "cd", "cq", "ncm", "ncd", "ncq")

    def __init__(self, ctx, verts, loop_off):
        verts = np.ascontiguousarray(verts, dtype=np.float64).reshape(-1, 3)
        loop_off = np.ascontiguousarray(loop_off, dtype=np.int64)
        h = _vp()
        with ctx.lock:
            _check(ctx.lib.lc_bh_forest_build(ctx.handle, _ptr(verts), _ptr(loop_off), len(loop_off) - 1,
                                              ctypes.byref(h)))
        self.ctx, self.handle = ctx, h
        L, M, N, lv = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
        _check(ctx.lib.lc_bh_forest_sizes(h, ctypes.byref(L), ctypes.byref(M), ctypes.byref(N), ctypes.byref(lv)))
        self.num_trees, self.num_segments, self.num_nodes, self.levels = L.value, M.value, N.value, lv.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                with self.ctx.lock:
                    self.ctx.lib.lc_bh_forest_free(self.ctx.handle, h)
            except Exception:
                pass
            self.handle = None

    def nodes(self, fields=FIELDS):
        """Host copies of node data, per-tree (reference) numbering."""
        L, M, N = self.num_trees, self.num_segments, self.num_nodes
        shapes = {"node_off": ((L + 1,), np.int64), "prim_order": ((M,), np.int64), "left": ((N,), np.int64),
                  "right": ((N,), np.int64), "start": ((N,), np.int64), "end": ((N,), np.int64),
                  "node_lo": ((N, 3), np.float64), "node_hi": ((N, 3), np.float64), "center": ((N, 3), np.float64),
                  "radius": ((N,), np.float64), "cm": ((N, 3), np.float64), "cd": ((N, 3, 3), np.float64),
                  "cq": ((N, 3, 3, 3), np.float64), "ncm": ((N,), np.float64), "ncd": ((N,), np.float64),
                  "ncq": ((N,), np.float64)}
        out = {f: np.empty(*shapes[f]) for f in fields}
        args = [_ptr(out.get(f)) for f in self.FIELDS]
        with self.ctx.lock:
            _check(self.ctx.lib.lc_bh_forest_nodes(self.ctx.handle, self.handle, *args))
        return out

    def far_field(self, node, other, other_node, quadrupole=True):
        out = ctypes.c_double(0.0)
        with self.ctx.lock:
            _check(self.ctx.lib.lc_bh_far_field(self.ctx.handle, self.handle, int(node), other.handle,
                                                int(other_node), int(bool(quadrupole)), ctypes.byref(out)))
        return out.value

    def eval(self, other, pairs, beta, quadrupole=True, k_const=1.0 / (4.0 * np.pi)):
        """Dual-tree Barnes-Hut sums for tree pairs (i in self, j in other): lam, e_est, visits."""
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        P = pairs.shape[0]
        beta = np.ascontiguousarray(np.broadcast_to(np.asarray(beta, dtype=np.float64), (P,)))
        lam = np.empty(P, dtype=np.float64)
        est = np.empty(P, dtype=np.float64)
        visits = ctypes.c_int64(0)
        with self.ctx.lock:
            _check(self.ctx.lib.lc_bh_eval(self.ctx.handle, self.handle, other.handle, _ptr(pairs), P, _ptr(beta),
                                           int(bool(quadrupole)), float(k_const), _ptr(lam), _ptr(est),
                                           ctypes.byref(visits)))
        return lam, est, visits.value


_ctx = {}
_ctx_lock = threading.Lock()


def context(device=None) -> Context:
    dev = default_device() if device is None else device
    with _ctx_lock:
        c = _ctx.get(dev)
        if c is None:
            c = Context(dev)
            _ctx[dev] = c
        return c
