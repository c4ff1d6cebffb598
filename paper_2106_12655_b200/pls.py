"""Potential link search — drop-in for linkcert.pls, computed on the GPU.

Reference: linkcert/pls.py:17-73.  Loop AABBs (unions of tight segment
boxes) and the closed-interval overlap sweep run in sm_100a kernels
(csrc/pls.cu); the result is the same sorted, deduplicated i<j pair set.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .geometry import CurveModel, ValidationError


class PairList:
    """Sorted, deduplicated (i, j) loop-index pairs with i < j (pls.py:17-45).

    Holds an int32 (P, 2) array (the device layout); the tuple view `pairs`
    is built on first access.
    """

    __slots__ = ("_array", "_pairs", "excluded")

    def __init__(self, pairs=(), excluded=frozenset()):
        norm = sorted({(int(i), int(j)) for i, j in pairs})
        for i, j in norm:
            if not i < j:
                raise ValidationError(f"pair ({i}, {j}) not ordered i < j")
        self._pairs = tuple(norm)
        self._array = np.asarray(norm, dtype=np.int32).reshape(-1, 2)
        self.excluded = _normalize_excluded(excluded)

    @classmethod
    def _from_sorted_array(cls, array, excluded=frozenset()):
        """Trusted constructor: `array` is already sorted, unique and i<j (device output)."""
        self = cls.__new__(cls)
        self._array = np.ascontiguousarray(array, dtype=np.int32).reshape(-1, 2)
        self._pairs = None
        self.excluded = _normalize_excluded(excluded)
        return self

    @property
    def pairs(self):
        if self._pairs is None:
            self._pairs = tuple(map(tuple, self._array.tolist()))
        return self._pairs

    @property
    def array(self):
        return self._array

    def __iter__(self):
        return iter(self.pairs)

    def __len__(self):
        return self._array.shape[0]

    def __eq__(self, other):
        if not isinstance(other, PairList):
            return NotImplemented
        return np.array_equal(self._array, other._array) and self.excluded == other.excluded

    def __hash__(self):
        return hash((self.pairs, self.excluded))

    def __repr__(self):
        return f"PairList(pairs={self.pairs!r}, excluded={self.excluded!r})"

    def loops_involved(self):
        return set(np.unique(self._array).tolist())


def _normalize_excluded(excluded):
    return frozenset((min(int(i), int(j)), max(int(i), int(j))) for i, j in excluded)


def excluded_keys(excluded):
    """Sorted unique uint64 keys (min<<32 | max) of an excluded-pair collection."""
    norm = _normalize_excluded(excluded)
    if not norm:
        return np.zeros(0, dtype=np.uint64)
    arr = np.array(sorted(norm), dtype=np.uint64).reshape(-1, 2)
    return np.unique((arr[:, 0] << np.uint64(32)) | arr[:, 1])


def upload(model: CurveModel, ctx=None, snapshot=None):
    """Stage the model's packed arrays on the device (boxes are derived per run)."""
    ctx = ctx or _native.context()
    snap = snapshot if snapshot is not None else model.snapshot()
    if snap.poly:       # the loops' own vertex arrays: 24 B/segment, gathered by the library
        ctx.upload_model_polyline_ptrs(snap.vptrs, snap.off)
    else:
        ctx.upload_model(*snap.packed())
    return ctx


def loop_boxes(model: CurveModel):
    """Per-loop AABB corners, unions of tight per-segment boxes (pls.py:48-56)."""
    ctx = upload(model)
    return ctx.loop_boxes()


def potential_link_search(model: CurveModel, excluded=()) -> PairList:
    """All loop pairs with overlapping AABBs, minus the excluded set (pls.py:59-73)."""
    if model.num_loops < 1:
        raise ValidationError("model has no loops")
    if model.num_loops == 1:
        return PairList((), excluded)
    ctx = upload(model)
    ctx.potential_link_search(excluded_keys(excluded))
    return PairList._from_sorted_array(ctx.get_pairs(), excluded)
