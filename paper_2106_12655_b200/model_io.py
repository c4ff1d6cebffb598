"""Canonical model serialization and digest — drop-in subset of linkcert.model_io.

Reference: linkcert/model_io.py:22-176.  Only what the verify path needs is
in scope: ParseError, model_to_dict and model_digest (SHA-256 of the
canonical json-curves document, called by compute_linking_matrix and
verify, certify.py:163,188).  File loading/saving is out of scope.
"""

from __future__ import annotations

import hashlib
import json
import math

import numpy as np

from . import _native
from .geometry import CurveModel, ValidationError


class ParseError(ValueError):
    """A model or certificate cannot be parsed (model_io.py:25-26)."""


def _num(x):
    x = float(x)
    if not math.isfinite(x):
        raise ValidationError("cannot serialize non-finite coordinate")
    return x


def model_to_dict(model: CurveModel, extra=None) -> dict:
    """Canonical json-curves dictionary (model_io.py:122-149)."""
    loops = []
    for loop in model.loops:
        plain = loop.is_polyline and np.all(loop.t[:, 0] == 0.0) and np.all(loop.t[:, 1] == 1.0)
        if plain:
            pts = loop.coeffs[:, 0]
            if not loop.closed:
                pts = np.vstack([pts, loop.end_points()[-1:]])
            if not np.all(np.isfinite(pts)):
                raise ValidationError("cannot serialize non-finite coordinate")
            loops.append({"type": "polyline", "closed": loop.closed, "points": pts.tolist()})
        else:
            loops.append({
                "type": "cubics",
                "closed": loop.closed,
                "segments": [
                    {"coeffs": [[_num(x) for x in row] for row in c], "t": [t0, t1]}
                    for c, (t0, t1) in zip(loop.coeffs, loop.t)
                ],
            })
    doc = {"loops": loops}
    if extra:
        doc.update(extra)
    return doc


def canonical_json(model: CurveModel):
    """Bytes of json.dumps(model_to_dict(model), sort_keys=True, separators=(",", ":")),
    formatted by the library's multithreaded writer (csrc/digest.cpp)."""
    coeffs, t, off = model.packed()
    closed = model.closed_flags()
    blob = _native.model_json(coeffs, t, off, None if closed.all() else closed)
    if blob is None:
        raise ValidationError("cannot serialize non-finite coordinate")
    return blob


def model_digest(model: CurveModel, snapshot=None) -> str:
    """SHA-256 hex digest of the canonical json-curves serialization (model_io.py:169-172).

    Formatting and hashing run in the library (csrc/digest.cpp) on all host
    cores with the GIL released, so callers can overlap it with GPU work.
    """
    coeffs, t, off, closed, _ = snapshot if snapshot is not None else model.snapshot()
    digest = _native.model_digest(coeffs, t, off, None if closed.all() else closed)
    if digest is None:
        raise ValidationError("cannot serialize non-finite coordinate")
    return digest


def model_digest_python(model: CurveModel) -> str:
    """Straight json.dumps restatement (cross-check for canonical_json in the tests)."""
    blob = json.dumps(model_to_dict(model), sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(blob.encode()).hexdigest()
