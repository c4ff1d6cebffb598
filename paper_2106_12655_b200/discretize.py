"""Adaptive homotopy-preserving spline -> polyline conversion, on the GPU.

Drop-in for linkcert.discretize (discretize.py:20-191): same parameters,
same error kinds, loops and messages.  The pass loop runs in sm_100a kernels
(csrc/discretize.cu) over packed SoA subsegment lists; the chords come back
as one packed float64 vertex array.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _native
from .geometry import MACHINE_EPS, CurveModel, PolylineLoop, ValidationError
from .pls import PairList, upload

ZERO_LENGTH_INPUT = "ZeroLengthInput"
CURVES_INTERSECT = "CurvesIntersect"
PASS_LIMIT_EXCEEDED = "PassLimitExceeded"


@dataclass
class DiscretizationParams:
    """discretize.py:25-40."""

    epsilon: float = MACHINE_EPS
    max_passes: int = 64
    max_subsegments: int = 1 << 22

    def __post_init__(self):
        if not self.epsilon > 0.0:
            raise ValueError("epsilon must be positive")
        if self.max_passes < 1:
            raise ValueError("max_passes must be >= 1")
        if self.max_subsegments < 1:
            raise ValueError("max_subsegments must be >= 1")


class DiscretizationError(Exception):
    """Refinement failed; `kind` names the failure, `loops` the offenders (discretize.py:43-49)."""

    def __init__(self, kind, loops, message):
        super().__init__(message)
        self.kind = kind
        self.loops = tuple(int(i) for i in loops)


_POLYLINE_MESSAGES = {
    1: "closed polyline needs >= 3 vertices",
    2: "polyline has non-finite vertices",
    3: "polyline has a zero-length segment",
}


def raise_for_failure(fail: _native.DiscretizeFailure, params: DiscretizationParams):
    """Map a device failure record onto the reference's exception and message."""
    k = fail.kind
    if k == _native.DISC_ZERO_LENGTH:
        raise DiscretizationError(ZERO_LENGTH_INPUT, fail.loops, "Input has zero-length segments.")
    if k == _native.DISC_CURVES_INTERSECT:
        a, b = fail.loops
        raise DiscretizationError(CURVES_INTERSECT, (a, b), f"Curves {a} and {b} intersect.")
    if k == _native.DISC_SUBSEG_BUDGET:
        (i,) = fail.loops
        raise DiscretizationError(
            PASS_LIMIT_EXCEEDED, (i,),
            f"loop {i} exceeded the {params.max_subsegments} subsegment refinement budget",
        )
    if k == _native.DISC_PASS_BUDGET:
        raise DiscretizationError(
            PASS_LIMIT_EXCEEDED, fail.loops,
            f"refinement did not settle within {params.max_passes} passes",
        )
    if k == _native.DISC_INVALID_POLYLINE:
        raise ValidationError(_POLYLINE_MESSAGES.get(fail.detail, "invalid polyline"))
    raise RuntimeError(f"unknown discretization failure {fail}")


def run_on_device(ctx, model: CurveModel, params: DiscretizationParams):
    """Discretize the model already uploaded to `ctx` with its staged pair list."""
    try:
        return ctx.discretize(model.xi, params.epsilon, params.max_passes, params.max_subsegments)
    except _native.DiscretizeFailure as fail:
        raise_for_failure(fail, params)


def split_polylines(verts, off):
    """Per-loop PolylineLoop views of one packed vertex array (validated on device)."""
    return [PolylineLoop._trusted(verts[off[k]:off[k + 1]]) for k in range(len(off) - 1)]


def discretize(model: CurveModel, pairs: PairList, params: DiscretizationParams | None = None):
    """Refine paired loops into link-equivalent closed polylines (discretize.py:112-191).

    Returns one PolylineLoop per input loop; raises DiscretizationError for
    degenerate input, intersecting paired curves or an exhausted budget.
    """
    params = params or DiscretizationParams()
    ctx = upload(model)
    arr = pairs.array if isinstance(pairs, PairList) else PairList(tuple(pairs)).array
    ctx.set_pairs(arr)
    run_on_device(ctx, model, params)
    verts, off = ctx.get_polylines()
    return split_polylines(verts, off)
