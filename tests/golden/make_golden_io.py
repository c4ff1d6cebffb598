"""Model-file golden vectors from the REFERENCE (linkcert/model_io.py), this container only.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_io.py

For models of tests/cases.py: SHA-256 of the file written by the reference's
save_json_curves.  For small hand-written files (stored inline): the
reference's load_model outcome (digest and xi, or the exception type and
message).  Writes tests/golden/golden_io.json.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import linkcert as ref  # noqa: E402
from linkcert import model_io as rio  # noqa: E402

import cases  # noqa: E402
from make_golden import to_ref  # noqa: E402

FILES = {
    "text_two_loops": ("polyline-text", "v 0 0 0\nv 1 0 0\nv 1 1 0\nv 0 1 0\n\nv 0.5 0.5 -1\nv 0.5 0.5 1\nv 0.6 2 0\n"),
    "text_bad_tag": ("polyline-text", "v 0 0 0\nw 1 0 0\nv 1 1 0\n"),
    "text_bad_number": ("polyline-text", "v 0 0 0\nv 1 x 0\nv 1 1 0\n"),
    "text_nan": ("polyline-text", "v 0 0 0\nv 1 nan 0\nv 1 1 0\n"),
    "json_mixed": ("json-curves", json.dumps({"loops": [
        {"type": "polyline", "points": [[0, 0, 0], [2, 0, 0], [2, 2, 0], [0, 2, 0]]},
        {"type": "catmullrom", "points": [[1, 1, -1], [1.2, 1, 1], [1, 3, 1], [0.8, 1, -1], [1.1, 0.5, 0]]},
        {"type": "cubics", "closed": True, "segments": [
            {"coeffs": [[5, 0, 0], [1, 0, 0], [0, 0, 0], [0, 0, 0]]},
            {"coeffs": [[6, 0, 0], [0, 1, 0], [0, 0, 0], [0, 0, 0]], "t": [0.0, 1.0]},
            {"coeffs": [[6, 1, 0], [-1, -1, 0], [0, 0, 0], [0, 0, 0]]}]},
        {"type": "polyline", "closed": False, "points": [[10, 0, 0], [11, 0, 0], [11, 1, 0]]}]})),
    "json_no_loops": ("json-curves", json.dumps({"curves": []})),
    "json_malformed": ("json-curves", "{\"loops\": [}"),
    "json_bad_type": ("json-curves", json.dumps({"loops": [{"type": "nurbs", "points": []}]})),
    "json_bad_points": ("json-curves", json.dumps({"loops": [{"type": "polyline", "points": [[0, 0], [1, 1]]}]})),
    "json_open_catmullrom": ("json-curves", json.dumps({"loops": [{"type": "catmullrom", "closed": False,
                                                                  "points": [[0, 0, 0], [1, 0, 0], [1, 1, 0]]}]})),
    "json_bad_coeffs": ("json-curves", json.dumps({"loops": [{"type": "cubics", "segments": [
        {"coeffs": [[0, 0, 0], [1, 0, 0]]}]}]})),
    "json_short_loop": ("json-curves", json.dumps({"loops": [{"type": "polyline", "points": [[0, 0, 0], [1, 0, 0]]}]})),
}


def main():
    out = {"saved": {}, "loaded": {}}
    with tempfile.TemporaryDirectory() as d:
        for name, model in cases.cert_models().items():
            if name in ("e4in1_32x32", "grid20", "unlinked200"):
                continue
            p = os.path.join(d, name + ".json")
            rio.save_json_curves(to_ref(model), p)
            out["saved"][name] = {"sha256": hashlib.sha256(Path(p).read_bytes()).hexdigest(),
                                  "fingerprint": cases.fingerprint(model)}
        for name, (fmt, text) in FILES.items():
            p = os.path.join(d, name)
            Path(p).write_text(text)
            try:
                m = ref.load_model(p, format=fmt)
                out["loaded"][name] = {"format": fmt, "text": text, "digest": ref.model_digest(m), "xi": m.xi,
                                       "num_loops": m.num_loops}
            except Exception as exc:  # noqa: BLE001
                msg = str(exc).replace(p, "<path>")
                out["loaded"][name] = {"format": fmt, "text": text, "error": type(exc).__name__, "message": msg}
    (HERE / "golden_io.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print(json.dumps({k: (v.get("error"), v.get("message")) for k, v in out["loaded"].items()}, indent=1))


if __name__ == "__main__":
    main()
