"""Curve / loop data model — host-side mirror of linkcert.geometry.

Same types, constructors, validation rules and exception types as the
reference (linkcert/geometry.py:14-360).  Everything numeric on the hot path
(tight boxes, PLS, discretization, Gauss sums) runs on the GPU through the
C-ABI; the host types here only hold float64 arrays.

B200-first addition: a CurveModel keeps one packed copy of all its loops
(coeffs (M, 4, 3), t (M, 2), loop offsets (L+1)) — the layout the device
pipeline consumes — built once and cached.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

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


class LoopGeometry:
    """Ordered chain of cubic segments, optionally closed (geometry.py:206-296)."""

    def __init__(self, coeffs, t=None, closed=True, control_points=None, xi_hint=None):
        coeffs = np.asarray(coeffs, dtype=np.float64)
        if coeffs.ndim != 3 or coeffs.shape[1:] != (4, 3):
            raise ValidationError("loop coeffs must be (m, 4, 3)")
        if not np.all(np.isfinite(coeffs)):
            raise ValidationError("loop has non-finite coefficients")
        m = coeffs.shape[0]
        t = np.tile(np.array([0.0, 1.0]), (m, 1)) if t is None else np.asarray(t, dtype=np.float64)
        if t.shape != (m, 2) or np.any(t[:, 0] >= t[:, 1]):
            raise ValidationError("bad segment parameter domains")
        self.coeffs = coeffs
        self.t = t
        self.closed = bool(closed)
        self.control_points = np.asarray(
            self.start_points() if control_points is None else control_points, dtype=np.float64
        )
        if closed and m < 3:
            raise ValidationError(f"closed loop needs >= 3 segments, got {m}")
        if xi_hint is None:
            xi_hint = float(np.mean(np.abs(self.control_points))) or 1.0
        starts, ends = self.start_points(), self.end_points()
        nxt = np.roll(starts, -1, axis=0) if closed else starts[1:]
        gaps = np.linalg.norm((ends if closed else ends[:-1]) - nxt, axis=1)
        if gaps.size and float(gaps.max()) > CONTINUITY_TOL * xi_hint:
            raise ValidationError(f"consecutive segments do not share endpoints (max gap {gaps.max():.3e})")

    @classmethod
    def _trusted(cls, coeffs, t, closed, control_points):
        """Construct without re-validation (arrays already validated in bulk)."""
        self = cls.__new__(cls)
        self.coeffs = coeffs
        self.t = t
        self.closed = closed
        self.control_points = control_points
        return self

    def __len__(self):
        return self.coeffs.shape[0]

    def start_points(self):
        return eval_cubics(self.coeffs, self.t[:, 0])

    def end_points(self):
        return eval_cubics(self.coeffs, self.t[:, 1])

    @property
    def is_polyline(self):
        return not np.any(self.coeffs[:, 2:])

    def boxes(self):
        return tight_boxes(self.coeffs, self.t[:, 0], self.t[:, 1])

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
        starts = verts if closed else verts[:-1]
        ends = np.roll(verts, -1, axis=0) if closed else verts[1:]
        coeffs = np.zeros((len(starts), 4, 3))
        coeffs[:, 0] = starts
        coeffs[:, 1] = ends - starts
        return LoopGeometry(coeffs, closed=closed, control_points=verts)

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

    # ---- B200 packed layout -------------------------------------------------
    def packed(self):
        """(coeffs (M,4,3), t (M,2), loop_off (L+1)) float64/int64, cached."""
        key = tuple(map(id, self.loops))
        cache = self.__dict__.get("_packed_cache")
        if cache is not None and cache[0] == key:
            return cache[1]
        if self.loops:
            from . import _native

            counts = np.fromiter((lp.coeffs.shape[0] for lp in self.loops), dtype=np.int64, count=len(self.loops))
            # page-locked: verify copies these to the device on every call
            coeffs = _native.pinned_empty((int(counts.sum()), 4, 3))
            np.concatenate([lp.coeffs for lp in self.loops], out=coeffs)
            t = _native.pinned_empty((int(counts.sum()), 2))
            np.concatenate([lp.t for lp in self.loops], out=t)
        else:
            counts = np.zeros(0, dtype=np.int64)
            coeffs = np.zeros((0, 4, 3))
            t = np.zeros((0, 2))
        off = np.zeros(len(counts) + 1, dtype=np.int64)
        np.cumsum(counts, out=off[1:])
        packed = (coeffs, t, off)
        self.__dict__["_packed_cache"] = (key, packed)
        self.__dict__.pop("_polyline_cache", None)
        return packed

    def closed_flags(self):
        """(L,) uint8 closedness of every loop, cached with the packed arrays."""
        return self._closed_of(self.packed()[0])

    def _closed_of(self, coeffs):
        cache = self.__dict__.get("_closed_cache")
        if cache is not None and cache[0] is coeffs:
            return cache[1]
        flags = np.fromiter((lp.closed for lp in self.loops), dtype=np.uint8, count=len(self.loops))
        self.__dict__["_closed_cache"] = (coeffs, flags)
        return flags

    def polyline_vertices(self):
        """(verts (M, 3), loop_off) when every loop is a plain closed polyline whose
        arrays are exactly LoopGeometry.from_polyline's (a1 = next - start bitwise,
        a2 = a3 = 0, t = [0, 1]) — then only the vertices need to reach the GPU.
        None otherwise.  Cached with the packed arrays."""
        return self._poly_of(*self.packed())

    def _poly_of(self, coeffs, t, off):
        cache = self.__dict__.get("_polyline_cache")
        if cache is not None and cache[0] is coeffs:
            return cache[1]
        result = None
        if len(off) > 1 and all(lp.closed for lp in self.loops) and np.all(np.diff(off) >= 1):
            nxt = np.arange(len(coeffs), dtype=np.int64) + 1
            nxt[off[1:] - 1] = off[:-1]
            a0 = coeffs[:, 0]
            if (not np.any(coeffs[:, 2:]) and np.all(t[:, 0] == 0.0) and np.all(t[:, 1] == 1.0)
                    and np.array_equal((a0[nxt] - a0).view(np.int64), coeffs[:, 1].view(np.int64))):
                from . import _native

                result = (_native.pinned_copy(a0), off)   # page-locked upload source
        self.__dict__["_polyline_cache"] = (coeffs, result)
        return result

    def snapshot(self):
        """(coeffs, t, loop_off, closed, polyline) of the current loops after a single
        cache check — what one verify / certificate call hands to the digest
        thread and to the device upload."""
        coeffs, t, off = self.packed()
        return coeffs, t, off, self._closed_of(coeffs), self._poly_of(coeffs, t, off)

    def snapshot_hint(self):
        """The cached snapshot if a cheap O(1) check (loop count, first and last loop
        identity) says the loops are unchanged, else None.  Only a head start: the
        caller still runs snapshot() and must discard work done on a stale hint."""
        cache = self.__dict__.get("_packed_cache")
        loops = self.loops
        if cache is None or not loops:
            return None
        key, (coeffs, t, off) = cache
        if len(key) != len(loops) or key[0] != id(loops[0]) or key[-1] != id(loops[-1]):
            return None
        closed = self.__dict__.get("_closed_cache")
        poly = self.__dict__.get("_polyline_cache")
        if closed is None or closed[0] is not coeffs or poly is None or poly[0] is not coeffs:
            return None
        return coeffs, t, off, closed[1], poly[1]

    @classmethod
    def from_polyline_arrays(cls, verts, offsets, closed=True):
        """Bulk constructor for closed polylines given as one (V,3) array + offsets.

        Equivalent to CurveModel([LoopGeometry.from_polyline(v) for v in
        split(verts)]) — same validation, same arrays, same xi — but checks
        every loop in one vectorized pass and fills the packed cache.
        """
        verts = np.ascontiguousarray(verts, dtype=np.float64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        if verts.ndim != 2 or verts.shape[1] != 3:
            raise ValidationError("polyline vertices must be (n, 3)")
        if not closed:
            raise ValidationError("bulk constructor supports closed loops only")
        if not np.all(np.isfinite(verts)):
            raise ValidationError("polyline has non-finite vertices")
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
        loops = [
            LoopGeometry._trusted(coeffs[off[k]:off[k + 1]], t[off[k]:off[k + 1]], True, verts[off[k]:off[k + 1]])
            for k in range(L)
        ]
        # xi exactly as compute_xi: sequential float accumulation of per-loop sums
        total = 0.0
        for s in sums.tolist():
            total += s
        xi = total / (3 * len(verts)) if len(verts) else 0.0
        model = cls(loops, xi=xi)
        model.__dict__["_packed_cache"] = (tuple(map(id, loops)), (coeffs, t, off))
        from . import _native

        model.__dict__["_polyline_cache"] = (coeffs, (_native.pinned_copy(verts), off))   # page-locked upload source
        model.__dict__["_closed_cache"] = (coeffs, np.ones(L, dtype=np.uint8))
        return model


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
    "Aabb", "CONTINUITY_TOL", "CubicSegment", "CurveModel", "LoopGeometry", "MACHINE_EPS", "PolylineLoop",
    "ValidationError", "catmull_rom_coeffs", "catmull_rom_to_cubics", "compute_xi", "eval_cubics",
    "split_cubic", "tight_aabb_of_cubic", "tight_boxes",
]

