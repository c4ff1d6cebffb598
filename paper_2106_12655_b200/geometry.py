"""Curve / loop data model — host-side mirror of linkcert.geometry.

Same types, constructors, validation rules and exception types as the
reference (linkcert/geometry.py:14-360).  Everything numeric on the hot path
(tight boxes, PLS, discretization, Gauss sums) runs on the GPU through the
C-ABI; the host types here only hold float64 arrays.

B200-first addition: a CurveModel hands the device pipeline and the digest a
ModelSnapshot of its loops — the loops' own vertex arrays (closed
from_polyline loops) or a packed copy (coeffs (M, 4, 3), t (M, 2), loop
offsets (L+1)) — cached while the loops are unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from operator import attrgetter, itemgetter
from struct import Struct

import numpy as np

# a closed from_polyline loop's vertex-array address and row count, packed (uint64,
# int64) so a snapshot joins every loop's record into one buffer
_pack_pn = Struct("<Qq").pack

MACHINE_EPS = np.finfo(np.float64).eps          # geometry.py:14
CONTINUITY_TOL = 1e-12                           # geometry.py:18


class ValidationError(ValueError):
    """Input geometry violates a structural invariant (geometry.py:21-22)."""


def _vec3(p, name="point"):
    v = np.asarray(p, dtype=np.float64)
    if v.shape != (3,):
        raise ValidationError(f"{name} must have 3 components, got shape {v.shape}")
    if not np.all(np.isfinite(v)):
        raise ValidationError(f"{name} has non-finite components: {v}")
    return v


def eval_cubics(coeffs, t):
    """Points of (m, 4, 3) monomial cubics at parameters t (m,) (geometry.py:107-110).

    Host helper for the data model; evaluation order a0 + a1 t + a2 t t + a3 t**3
    is the one the device kernels reproduce.
    """
    t = np.asarray(t, dtype=np.float64)[:, None]
    return coeffs[:, 0] + coeffs[:, 1] * t + coeffs[:, 2] * t * t + coeffs[:, 3] * t**3


def tight_boxes(coeffs, t_lo, t_hi):
    """Tight AABBs (lo, hi) of monomial cubics over their domains, on the GPU.

    Reference: geometry.py:113-152.  Computed by the sm_100a kernel behind
    lc_model_upload/lc_loop_boxes' segment stage (no CPU fallback).
    """
    from . import _native

    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(-1, 4, 3)
    m = coeffs.shape[0]
    t = np.empty((m, 2))
    t[:, 0] = np.broadcast_to(np.asarray(t_lo, dtype=np.float64), (m,))
    t[:, 1] = np.broadcast_to(np.asarray(t_hi, dtype=np.float64), (m,))
    return _native.context().tight_boxes(coeffs, t)


@dataclass(frozen=True)
class CubicSegment:
    """p(t) = a0 + a1 t + a2 t^2 + a3 t^3 over [t_lo, t_hi] (geometry.py:34-74)."""

    coeffs: np.ndarray
    t_lo: float = 0.0
    t_hi: float = 1.0

    def __post_init__(self):
        c = np.asarray(self.coeffs, dtype=np.float64)
        if c.shape != (4, 3):
            raise ValidationError(f"cubic coeffs must be (4, 3), got {c.shape}")
        if not np.all(np.isfinite(c)):
            raise ValidationError("cubic coefficients must be finite")
        if not (0.0 <= self.t_lo < self.t_hi <= 1.0):
            raise ValidationError(f"bad parameter domain [{self.t_lo}, {self.t_hi}]")
        object.__setattr__(self, "coeffs", c)

    def point(self, t):
        t = np.asarray(t, dtype=np.float64)
        a0, a1, a2, a3 = self.coeffs
        return a0 + np.multiply.outer(t, a1) + np.multiply.outer(t * t, a2) + np.multiply.outer(t * t * t, a3)

    @property
    def start(self):
        return self.point(self.t_lo)

    @property
    def end(self):
        return self.point(self.t_hi)

    @staticmethod
    def straight(p, q):
        p, q = _vec3(p), _vec3(q)
        z = np.zeros(3)
        return CubicSegment(np.array([p, q - p, z, z]))


@dataclass(frozen=True)
class Aabb:
    """Closed axis-aligned box (geometry.py:77-104)."""

    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        lo, hi = _vec3(self.min, "box min"), _vec3(self.max, "box max")
        if np.any(lo > hi):
            raise ValidationError(f"box min {lo} exceeds max {hi}")
        object.__setattr__(self, "min", lo)
        object.__setattr__(self, "max", hi)

    def overlaps(self, other):
        return bool(np.all(self.min <= other.max) and np.all(other.min <= self.max))

    def contains(self, p, slack=0.0):
        p = np.asarray(p, dtype=np.float64)
        return bool(np.all(p >= self.min - slack) and np.all(p <= self.max + slack))

    @property
    def diameter(self):
        return float(np.linalg.norm(self.max - self.min))

    @property
    def center(self):
        return 0.5 * (self.min + self.max)


def tight_aabb_of_cubic(seg: CubicSegment) -> Aabb:
    lo, hi = tight_boxes(seg.coeffs[None], np.array([seg.t_lo]), np.array([seg.t_hi]))
    return Aabb(lo[0], hi[0])


def split_cubic(seg: CubicSegment):
    mid = 0.5 * (seg.t_lo + seg.t_hi)
    return CubicSegment(seg.coeffs, seg.t_lo, mid), CubicSegment(seg.coeffs, mid, seg.t_hi)


def catmull_rom_coeffs(pts):
    """Monomial coefficients (n, 4, 3) of a closed uniform Catmull-Rom cycle (geometry.py:189-203)."""
    p0 = np.asarray(pts, dtype=np.float64)
    p1 = np.roll(p0, -1, axis=0)
    m0 = 0.5 * (p1 - np.roll(p0, 1, axis=0))
    m1 = 0.5 * (np.roll(p0, -2, axis=0) - p0)
    out = np.empty((len(p0), 4, 3))
    out[:, 0] = p0
    out[:, 1] = m0
    out[:, 2] = -3.0 * p0 + 3.0 * p1 - 2.0 * m0 - m1
    out[:, 3] = 2.0 * p0 - 2.0 * p1 + m0 + m1
    return out


def catmull_rom_to_cubics(control_points) -> list[CubicSegment]:
    pts = np.asarray(control_points, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ValidationError("control points must be an (n, 3) array")
    if not np.all(np.isfinite(pts)):
        raise ValidationError("control points must be finite")
    if len(pts) < 4:
        raise ValidationError(f"need at least 4 control points, got {len(pts)}")
    if np.any(np.all(pts == np.roll(pts, -1, axis=0), axis=1)):
        raise ValidationError("duplicate adjacent control points (zero tangent)")
    return [CubicSegment(c) for c in catmull_rom_coeffs(pts)]


_EPOCH = [0]   # bumped by every attribute assignment on any LoopGeometry (model snapshot validity)


def _owned(a, frozen=True):
    """Owned, C-contiguous float64 copy of `a`, read-only: a loop's arrays cannot
    change under a cached model snapshot (in-place edits raise; reassignment of
    the attribute is seen by the loop's stamp)."""
    out = np.array(a, dtype=np.float64, order="C")
    if frozen:
        out.setflags(write=False)
    return out


def _loop_attr(name, conv):
    def get(self):
        return self.__dict__[name]

    def put(self, value):
        d = self.__dict__
        d[name] = conv(value)
        d["_pv"] = None                 # no longer known to be a plain from_polyline loop
        _EPOCH[0] += 1
        d["_stamp"] = _EPOCH[0]

    return property(get, put)


class LoopGeometry:
    """Ordered chain of cubic segments, optionally closed (geometry.py:206-296).

    B200-first ownership: the loop keeps owned, read-only copies of its arrays
    (the reference aliases the caller's arrays, geometry.py:225-230), so a
    CurveModel can cache what it uploads and hashes.  Reassigning an attribute
    (loop.coeffs = ...) is tracked; editing an array in place raises ValueError.
    A closed loop built by from_polyline remembers its vertex array (with its
    address and row count, `_pv`): a model of such loops reaches the GPU and the
    digest as vertices only (24 B/segment).
    """

    coeffs = _loop_attr("_coeffs", _owned)
    t = _loop_attr("_t", _owned)
    control_points = _loop_attr("_cp", _owned)
    closed = _loop_attr("_closed", bool)

    def __init__(self, coeffs, t=None, closed=True, control_points=None, xi_hint=None):
        coeffs = _owned(coeffs, frozen=False)
        t = None if t is None else _owned(t, frozen=False)
        cp = None if control_points is None else _owned(control_points, frozen=False)
        self._setup(coeffs, t, closed, cp, xi_hint)

    def _setup(self, coeffs, t, closed, cp, xi_hint, pv=None):
        """Validate (geometry.py:216-240) and take ownership of already-owned arrays."""
        if coeffs.ndim != 3 or coeffs.shape[1:] != (4, 3):
            raise ValidationError("loop coeffs must be (m, 4, 3)")
        if not np.all(np.isfinite(coeffs)):
            raise ValidationError("loop has non-finite coefficients")
        m = coeffs.shape[0]
        if t is None:
            t = np.empty((m, 2))
            t[:, 0] = 0.0
            t[:, 1] = 1.0
        if t.shape != (m, 2) or np.any(t[:, 0] >= t[:, 1]):
            raise ValidationError("bad segment parameter domains")
        if cp is None:
            cp = eval_cubics(coeffs, t[:, 0])
        for a in (coeffs, t, cp):
            a.setflags(write=False)
        d = self.__dict__
        d["_coeffs"], d["_t"], d["_closed"], d["_cp"] = coeffs, t, bool(closed), cp
        d["_pv"] = pv
        d["_stamp"] = 0
        if closed and m < 3:
            raise ValidationError(f"closed loop needs >= 3 segments, got {m}")
        if xi_hint is None:
            xi_hint = float(np.mean(np.abs(cp))) or 1.0
        starts, ends = self.start_points(), self.end_points()
        nxt = np.roll(starts, -1, axis=0) if closed else starts[1:]
        gaps = np.linalg.norm((ends if closed else ends[:-1]) - nxt, axis=1)
        if gaps.size and float(gaps.max()) > CONTINUITY_TOL * xi_hint:
            raise ValidationError(f"consecutive segments do not share endpoints (max gap {gaps.max():.3e})")

    @classmethod
    def _view(cls, coeffs, t, verts, ptr):
        """A closed from_polyline loop over views of a validated read-only block."""
        self = cls.__new__(cls)
        d = self.__dict__
        d["_coeffs"], d["_t"], d["_closed"], d["_cp"] = coeffs, t, True, verts
        d["_pv"] = (verts, _pack_pn(ptr, verts.shape[0]))
        d["_stamp"] = 0
        return self

    def __len__(self):
        return self._coeffs.shape[0]

    def start_points(self):
        return eval_cubics(self._coeffs, self._t[:, 0])

    def end_points(self):
        return eval_cubics(self._coeffs, self._t[:, 1])

    @property
    def is_polyline(self):
        return not np.any(self._coeffs[:, 2:])

    def boxes(self):
        return tight_boxes(self._coeffs, self._t[:, 0], self._t[:, 1])

    def aabb(self) -> Aabb:
        lo, hi = self.boxes()
        return Aabb(lo.min(axis=0), hi.max(axis=0))

    @staticmethod
    def from_polyline(vertices, closed=True):
        verts = np.asarray(vertices, dtype=np.float64)
        if verts.ndim != 2 or verts.shape[1] != 3:
            raise ValidationError("polyline vertices must be (n, 3)")
        if not np.all(np.isfinite(verts)):
            raise ValidationError("polyline has non-finite vertices")
        verts = _owned(verts, frozen=False)
        starts = verts if closed else verts[:-1]
        ends = np.roll(verts, -1, axis=0) if closed else verts[1:]
        coeffs = np.zeros((len(starts), 4, 3))
        coeffs[:, 0] = starts
        coeffs[:, 1] = ends - starts
        loop = LoopGeometry.__new__(LoopGeometry)
        pv = (verts, _pack_pn(verts.ctypes.data, len(verts))) if closed and len(verts) else None
        loop._setup(coeffs, None, closed, verts, None, pv)
        return loop

    @staticmethod
    def from_segments(segments, closed=True):
        coeffs = np.stack([s.coeffs for s in segments])
        t = np.array([[s.t_lo, s.t_hi] for s in segments])
        return LoopGeometry(coeffs, t, closed=closed)

    @staticmethod
    def from_catmull_rom(control_points):
        pts = np.asarray(control_points, dtype=np.float64)
        loop = LoopGeometry.from_segments(catmull_rom_to_cubics(pts), closed=True)
        loop.control_points = pts
        return loop


def _loop_abs_sums(flat_abs, counts):
    """Per-loop float(np.sum(|pts|)) with numpy's own (pairwise) summation."""
    out = np.empty(len(counts))
    if len(counts) and np.all(counts == counts[0]):
        # rows of equal length reduce exactly like np.sum of each contiguous row
        out[:] = flat_abs.reshape(len(counts), -1).sum(axis=1)
        return out
    pos = 0
    for k, c in enumerate(counts):
        out[k] = float(np.sum(flat_abs[pos:pos + c]))
        pos += c
    return out


def compute_xi(loops):
    """Average |coordinate| over all control points (geometry.py:315-323)."""
    total = 0.0
    count = 0
    for loop in loops:
        pts = loop.control_points
        total += float(np.sum(np.abs(pts)))
        count += pts.size
    return total / count if count else 0.0


_get_pv, _item1 = attrgetter("_pv"), itemgetter(1)
_PIECE = 1024   # loops per piece of a streamed snapshot


class ModelSnapshot:
    """What one certificate / verify call hands to the digest thread and to the
    device upload, taken after one validity check of the model's loops.

    poly: every loop is a closed from_polyline loop -> `vptrs` (L) addresses of
    the loops' own vertex arrays (kept alive by `vrefs`) and `off` (L+1) reach
    the library directly (lc_model_upload_polyline_ptrs / lc_model_digest_polylines:
    no host-side packing).  Otherwise `packed()` = (coeffs (M,4,3), t (M,2), off)
    in page-locked memory.
    """

    __slots__ = ("key", "epoch", "poly", "off", "closed", "vptrs", "vrefs", "ready", "_packed")

    def __init__(self, loops, epoch, on_start=None):
        self.key = tuple(loops)
        self.epoch = epoch
        self._packed = None
        self.ready = None
        L = len(self.key)
        if on_start is not None and L > 2 * _PIECE and self._stream(on_start):
            return
        # two C-level passes over the loops: their (vertices, packed address + rows)
        # and the packed records joined into one buffer (~0.07 us per loop)
        pv = list(map(_get_pv, self.key))
        try:
            blob = b"".join(map(_item1, pv))       # TypeError: some loop is not a closed from_polyline loop
            self.poly = L > 0
        except TypeError:
            self.poly = False
        self.off = np.zeros(L + 1, dtype=np.int64)
        if self.poly:
            pn = np.frombuffer(blob, dtype=np.uint64).reshape(L, 2)
            self.vrefs = pv                        # keeps the vertex arrays alive while their addresses are used
            self.vptrs = np.ascontiguousarray(pn[:, 0])
            np.cumsum(pn[:, 1].view(np.int64), out=self.off[1:])
            self.closed = np.ones(L, dtype=np.uint8)
        else:
            self.vrefs = self.vptrs = None
            if L:
                np.cumsum(np.fromiter((len(lp) for lp in self.key), dtype=np.int64, count=L), out=self.off[1:])
            self.closed = np.fromiter((lp.closed for lp in self.key), dtype=np.uint8, count=L)

    def _stream(self, on_start):
        """A poly snapshot built piece by piece: after the first piece `on_start(self)`
        may hand vptrs / off / ready to a streamed digest, which formats and hashes
        loops [0, ready[0]) while the rest are walked.  False (and ready[0] = -1,
        aborting a started stream) when some loop is not a closed from_polyline loop."""
        key, L = self.key, len(self.key)
        self.vptrs = np.zeros(L, dtype=np.uint64)
        self.off = np.zeros(L + 1, dtype=np.int64)
        self.ready = np.zeros(1, dtype=np.int64)
        self.vrefs = []
        started = False
        try:
            for a in range(0, L, _PIECE):
                pv = list(map(_get_pv, key[a:a + _PIECE]))
                try:
                    blob = b"".join(map(_item1, pv))
                except TypeError:
                    return False
                n = len(pv)
                pn = np.frombuffer(blob, dtype=np.uint64).reshape(n, 2)
                self.vptrs[a:a + n] = pn[:, 0]
                part = self.off[a + 1:a + n + 1]
                np.cumsum(pn[:, 1].view(np.int64), out=part)
                part += self.off[a]
                self.vrefs.extend(pv)
                self.ready[0] = a + n         # published after the loops' entries (x86 store order)
                if not started:
                    on_start(self)
                    started = True
            self.poly = True
            self.closed = np.ones(L, dtype=np.uint8)
            return True
        finally:
            if self.ready[0] != L:
                self.ready[0] = -1

    def valid_for(self, loops, epoch):
        if self.key != tuple(loops):          # identity per element (LoopGeometry has no __eq__)
            return False
        if self.epoch != epoch:
            if any(lp._stamp > self.epoch for lp in self.key):
                return False
            self.epoch = epoch
        return True

    def packed(self):
        """(coeffs (M,4,3), t (M,2), loop_off (L+1)), page-locked, built on first use."""
        if self._packed is None:
            M = int(self.off[-1])
            if M:
                from . import _native

                coeffs = _native.pinned_empty((M, 4, 3))
                np.concatenate([lp.coeffs for lp in self.key], out=coeffs)
                t = _native.pinned_empty((M, 2))
                np.concatenate([lp.t for lp in self.key], out=t)
            else:
                coeffs, t = np.zeros((0, 4, 3)), np.zeros((0, 2))
            self._packed = (coeffs, t, self.off)
        return self._packed

    def vertices(self):
        """Packed (M, 3) vertices of a poly snapshot (a host copy; tests / tools)."""
        return np.concatenate([p[0] for p in self.vrefs]) if self.vrefs else np.zeros((0, 3))


@dataclass
class CurveModel:
    """A collection of loops plus the model coordinate scale xi (geometry.py:299-312)."""

    loops: list = field(default_factory=list)
    xi: float = 0.0

    def __post_init__(self):
        if self.loops and self.xi == 0.0:
            self.xi = compute_xi(self.loops)
        if self.loops and not self.xi > 0.0:
            raise ValidationError("model coordinate magnitude must be positive")

    @property
    def num_loops(self):
        return len(self.loops)

    # ---- B200 snapshot of the loops -------------------------------------------
    def snapshot(self, on_start=None) -> ModelSnapshot:
        """The loops as the device upload and the digest consume them.  Cached
        while the loop list holds the same objects and none of them had an
        attribute reassigned (their arrays are read-only); O(L) to check.
        on_start: see ModelSnapshot._stream (called only when a new snapshot of
        closed polylines is built)."""
        epoch = _EPOCH[0]
        snap = self.__dict__.get("_snapshot")
        if snap is not None and snap.valid_for(self.loops, epoch):
            return snap
        snap = ModelSnapshot(self.loops, epoch, on_start)
        self.__dict__["_snapshot"] = snap
        return snap

    def packed(self):
        """(coeffs (M,4,3), t (M,2), loop_off (L+1)) float64/int64 of the current loops."""
        return self.snapshot().packed()

    def closed_flags(self):
        """(L,) uint8 closedness of every loop."""
        return self.snapshot().closed

    def polyline_vertices(self):
        """(verts (M, 3), loop_off) when every loop is a closed from_polyline loop
        (only the vertices reach the GPU), else None."""
        snap = self.snapshot()
        return (snap.vertices(), snap.off) if snap.poly else None

    @classmethod
    def from_polyline_arrays(cls, verts, offsets, closed=True):
        """Bulk constructor for closed polylines given as one (V,3) array + offsets.

        Equivalent to CurveModel([LoopGeometry.from_polyline(v) for v in
        split(verts)]) — same validation, same arrays, same xi — but checks
        every loop in one vectorized pass; the loops are read-only views of one
        owned block.
        """
        verts = np.asarray(verts, dtype=np.float64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        if verts.ndim != 2 or verts.shape[1] != 3:
            raise ValidationError("polyline vertices must be (n, 3)")
        if not closed:
            raise ValidationError("bulk constructor supports closed loops only")
        if not np.all(np.isfinite(verts)):
            raise ValidationError("polyline has non-finite vertices")
        verts = _owned(verts, frozen=False)
        L = len(off) - 1
        counts = np.diff(off)
        if np.any(counts < 3):
            raise ValidationError("closed loop needs >= 3 segments")
        # next vertex within each loop (wrapping)
        idx = np.arange(len(verts), dtype=np.int64) + 1
        idx[off[1:] - 1] = off[:-1]
        nxt = verts[idx]
        coeffs = np.zeros((len(verts), 4, 3))
        coeffs[:, 0] = verts
        coeffs[:, 1] = nxt - verts
        t = np.zeros((len(verts), 2))
        t[:, 1] = 1.0
        # continuity: |(a0 + a1) - next start| <= tol * mean|pts| per loop
        ends = coeffs[:, 0] + coeffs[:, 1]
        gaps = np.linalg.norm(ends - nxt, axis=1)
        absv = np.abs(verts).reshape(-1)
        sums = _loop_abs_sums(absv, counts * 3)
        means = sums / (counts * 3)
        hint = np.where(means == 0.0, 1.0, means)
        gmax = np.maximum.reduceat(gaps, off[:-1]) if L else np.zeros(0)
        if np.any(gmax > CONTINUITY_TOL * hint):
            raise ValidationError("consecutive segments do not share endpoints")
        for a in (verts, coeffs, t):
            a.setflags(write=False)
        base = verts.ctypes.data
        ptrs = (base + 24 * off[:-1]).tolist()
        loops = [LoopGeometry._view(coeffs[off[k]:off[k + 1]], t[off[k]:off[k + 1]], verts[off[k]:off[k + 1]],
                                    ptrs[k])
                 for k in range(L)]
        # xi exactly as compute_xi: sequential float accumulation of per-loop sums
        total = 0.0
        for s in sums.tolist():
            total += s
        xi = total / (3 * len(verts)) if len(verts) else 0.0
        return cls(loops, xi=xi)


class PolylineLoop:
    """Closed vertex cycle; segment i runs vertex i -> i+1, wrapping (geometry.py:326-360)."""

    def __init__(self, vertices, xi_hint=None):
        verts = np.ascontiguousarray(vertices, dtype=np.float64)
        if verts.ndim != 2 or verts.shape[1] != 3:
            raise ValidationError("vertices must be (n, 3)")
        if len(verts) < 3:
            raise ValidationError("closed polyline needs >= 3 vertices")
        if not np.all(np.isfinite(verts)):
            raise ValidationError("polyline has non-finite vertices")
        seglen = np.linalg.norm(np.roll(verts, -1, axis=0) - verts, axis=1)
        scale = xi_hint if xi_hint else float(np.mean(np.abs(verts))) or 1.0
        if float(seglen.min()) <= MACHINE_EPS * scale:
            raise ValidationError("polyline has a zero-length segment")
        self.vertices = verts

    @classmethod
    def _trusted(cls, vertices):
        """Wrap device-validated vertices (the GPU already ran the checks above)."""
        self = cls.__new__(cls)
        self.vertices = vertices
        return self

    def __len__(self):
        return len(self.vertices)

    @property
    def closed_vertices(self):
        return np.vstack([self.vertices, self.vertices[:1]])

    def reversed(self):
        return PolylineLoop(self.vertices[::-1].copy())

    def total_length(self):
        return float(np.sum(np.linalg.norm(np.roll(self.vertices, -1, axis=0) - self.vertices, axis=1)))

    def aabb(self) -> Aabb:
        return Aabb(self.vertices.min(axis=0), self.vertices.max(axis=0))


__all__ = [
    "Aabb", "CONTINUITY_TOL", "CubicSegment", "CurveModel", "LoopGeometry", "MACHINE_EPS", "ModelSnapshot",
    "PolylineLoop",
    "ValidationError", "catmull_rom_coeffs", "catmull_rom_to_cubics", "compute_xi", "eval_cubics",
    "split_cubic", "tight_aabb_of_cubic", "tight_boxes",
]

