"""Model files, canonical serialization and digest — drop-in for linkcert.model_io.

Reference: linkcert/model_io.py:1-176.  The digest (SHA-256 of the canonical
json-curves document, called by compute_linking_matrix and verify,
certify.py:163,188) is formatted and hashed by the library (csrc/digest.cpp);
the file formats feeding the path are read and written here:

* json-curves: {"loops": [{"type": "polyline" | "catmullrom" | "cubics",
  "closed": bool, "points": [[x, y, z], ...]}]}; "cubics" loops carry
  "segments": [{"coeffs": 4 x 3, "t": [lo, hi]}] instead of "points".
* polyline-text: "v x y z" lines, a blank line closes a loop.
"""

from __future__ import annotations

import hashlib
import json
import math

import numpy as np

from . import _native
from .geometry import CurveModel, LoopGeometry, ValidationError, compute_xi


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
    snap = model.snapshot()
    coeffs, t, off = snap.packed()
    closed = snap.closed
    blob = _native.model_json(coeffs, t, off, None if closed.all() else closed)
    if blob is None:
        raise ValidationError("cannot serialize non-finite coordinate")
    return blob


def model_digest(model: CurveModel, snapshot=None, nthreads=0) -> str:
    """SHA-256 hex digest of the canonical json-curves serialization (model_io.py:169-172).

    Formatting and hashing run in the library (csrc/digest.cpp) on all host
    cores with the GIL released, so callers can overlap it with GPU work.
    """
    snap = snapshot if snapshot is not None else model.snapshot()
    if snap.poly:     # closed from_polyline loops: straight from their vertex arrays
        digest = _native.model_digest_polylines(snap.vptrs, snap.off, nthreads)
    else:
        coeffs, t, off = snap.packed()
        closed = snap.closed
        digest = _native.model_digest(coeffs, t, off, None if closed.all() else closed, nthreads)
    if digest is None:
        raise ValidationError("cannot serialize non-finite coordinate")
    return digest


def model_digest_python(model: CurveModel) -> str:
    """Straight json.dumps restatement (cross-check for canonical_json in the tests)."""
    blob = json.dumps(model_to_dict(model), sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(blob.encode()).hexdigest()


# ---- model files (model_io.py:29-119, 160-176) ------------------------------

def load_model(path, format="json-curves") -> CurveModel:
    readers = {"json-curves": load_json_curves, "polyline-text": load_polyline_text}
    if format not in readers:
        raise ParseError(f"unknown model format: {format!r}")
    return readers[format](path)


def load_json_curves(path) -> CurveModel:
    with open(path) as f:
        try:
            doc = json.load(f)
        except json.JSONDecodeError as exc:
            raise ParseError(f"malformed JSON in {path}: {exc}") from None
    return model_from_dict(doc)


def model_from_dict(doc) -> CurveModel:
    """CurveModel of a json-curves document; errors name the offending loop."""
    if not isinstance(doc, dict) or "loops" not in doc:
        raise ParseError("json-curves file must be an object with a 'loops' key")
    loops = []
    for idx, entry in enumerate(doc["loops"]):
        try:
            loops.append(_loop_from_entry(entry))
        except ValidationError as exc:
            raise ValidationError(f"loop {idx}: {exc}") from None
        except (ParseError, KeyError, TypeError, ValueError) as exc:
            raise ParseError(f"loop {idx}: {exc}") from None
    return CurveModel(loops)


def _xyz_rows(raw):
    pts = np.asarray(raw, dtype=np.float64)
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ParseError("points must be a list of [x, y, z] triples")
    if not np.isfinite(pts).all():
        raise ValidationError("points contain NaN or Inf")
    return pts


def _loop_from_entry(entry):
    kind = entry.get("type", "polyline")
    closed = bool(entry.get("closed", True))
    if kind == "polyline":
        return LoopGeometry.from_polyline(_xyz_rows(entry["points"]), closed=closed)
    if kind == "catmullrom":
        if not closed:
            raise ParseError("catmullrom loops must be closed")
        return LoopGeometry.from_catmull_rom(_xyz_rows(entry["points"]))
    if kind == "cubics":
        segs = entry["segments"]
        coeffs = [np.asarray(sg["coeffs"], dtype=np.float64) for sg in segs]
        for c in coeffs:
            if c.shape != (4, 3):
                raise ParseError(f"cubic coeffs must be 4x3, got {c.shape}")
        t = np.asarray([sg.get("t", [0.0, 1.0]) for sg in segs], dtype=np.float64)
        return LoopGeometry(np.stack(coeffs), t, closed=closed)
    raise ParseError(f"unknown loop type {kind!r}")


def load_polyline_text(path) -> CurveModel:
    loops, rows = [], []

    def close_block(where):
        pts = np.asarray(rows, dtype=np.float64)
        if not np.isfinite(pts).all():
            raise ValidationError(f"loop ending at line {where} has non-finite vertices")
        loops.append(LoopGeometry.from_polyline(pts, closed=True))
        rows.clear()

    with open(path) as f:
        for lineno, raw in enumerate(f, 1):
            line = raw.strip()
            if not line:
                if rows:
                    close_block(lineno)
                continue
            fields = line.split()
            if len(fields) != 4 or fields[0] != "v":
                raise ParseError(f"{path}:{lineno}: expected 'v x y z', got {line!r}")
            try:
                rows.append([float(x) for x in fields[1:]])
            except ValueError:
                raise ParseError(f"{path}:{lineno}: bad coordinate in {line!r}") from None
    if rows:
        close_block("eof")
    return CurveModel(loops)


def save_json_curves(model: CurveModel, path, extra=None):
    """json.dump(model_to_dict(model, extra), sort_keys=True) plus a newline.  Without
    `extra` the bytes come from the library's canonical writer with json.dump's
    default separators restored (every ',' and ':' of that document is structural)."""
    if extra:
        with open(path, "w") as f:
            json.dump(model_to_dict(model, extra=extra), f, sort_keys=True)
            f.write("\n")
        return
    blob = bytes(canonical_json(model)).replace(b",", b", ").replace(b":", b": ")
    with open(path, "wb") as f:
        f.write(blob)
        f.write(b"\n")


def recompute_xi(model: CurveModel) -> float:
    return compute_xi(model.loops)
