"""Gauss linking integral by exact segment-pair summation — on the GPU.

Drop-in for linkcert.direct (direct.py:137-166).  Both reference variants run
on the sm_100a Gauss-sum kernel (csrc/gauss.cu):
* "atan" (one signed-solid-angle arctangent pair per segment pair,
  direct.py:19-65) in the arithmetic form selected by LINKCERT_GAUSS_MODE
  (phase | atan | ref, default phase); all three agree with the reference to
  ~1e-14;
* "anglesum" (_link_angle_sum, direct.py:68-134) as the reference computes it:
  GAUSS_ANGLESUM, one lane per outer segment walking the inner segments in
  order with the reference's normalized phase product and crossing counts.
"""

from __future__ import annotations

import os

import numpy as np

from . import _native

VARIANTS = ("atan", "anglesum")


def gauss_mode():
    name = os.environ.get("LINKCERT_GAUSS_MODE", "phase").lower()
    try:
        return _native.GAUSS_MODES[name]
    except KeyError:
        raise ValueError(f"LINKCERT_GAUSS_MODE must be one of {sorted(_native.GAUSS_MODES)}, got {name!r}") from None


def ds_mode(variant="atan"):
    """Gauss-kernel mode of a direct-summation variant (KernelChoice.ds_variant)."""
    if variant == "anglesum":
        return _native.GAUSS_ANGLESUM
    if variant != "atan":
        raise ValueError(f"unknown direct-summation variant {variant!r}")
    return gauss_mode()


def _vertices(loop):
    verts = loop.vertices if hasattr(loop, "vertices") else np.asarray(loop, dtype=np.float64)
    return np.ascontiguousarray(verts, dtype=np.float64)


def segment_pair_lambda(l_j, l_j1, k_i, k_i1) -> float:
    """Linking contribution of one segment pair, signed-solid-angle form (direct.py:137-146)."""
    quad = np.concatenate([np.asarray(v, dtype=np.float64).reshape(3) for v in (l_j, l_j1, k_i, k_i1)])
    return float(_native.context().segment_pair_lambda(quad)[0])


def link_direct(loop1, loop2, variant="atan") -> float:
    """Real-valued linking number of two closed polylines (direct.py:149-161)."""
    mode = ds_mode(variant)
    return float(_native.context().link_direct(_vertices(loop1), _vertices(loop2), mode))
