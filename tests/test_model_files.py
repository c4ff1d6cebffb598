"""Model files (linkcert/model_io.py:29-176) against the reference's own
outputs (tests/golden/golden_io.json, make_golden_io.py): save_json_curves
writes byte-identical files; load_model reproduces the reference's models
(digest, xi) and its exceptions and messages.  CPU only (host code)."""

import hashlib
import json
from pathlib import Path

import pytest

import cases
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import model_io
from paper_2106_12655_b200.geometry import ValidationError

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "golden_io.json").read_text())


@pytest.mark.parametrize("name", sorted(GOLDEN["saved"]))
def test_save_json_curves_bytes(tmp_path, name):
    g = GOLDEN["saved"][name]
    model = cases.cert_models()[name]
    assert cases.fingerprint(model) == g["fingerprint"]
    p = tmp_path / "m.json"
    lc.save_json_curves(model, p)
    assert hashlib.sha256(p.read_bytes()).hexdigest() == g["sha256"]
    back = lc.load_model(p)
    assert lc.model_digest(back) == lc.model_digest(model) and back.xi == model.xi


@pytest.mark.parametrize("name", sorted(GOLDEN["loaded"]))
def test_load_model_matches_reference(tmp_path, name):
    g = GOLDEN["loaded"][name]
    p = tmp_path / name
    p.write_text(g["text"])
    if "error" in g:
        exc = {"ParseError": model_io.ParseError, "ValidationError": ValidationError}[g["error"]]
        with pytest.raises(exc) as info:
            lc.load_model(p, format=g["format"])
        assert type(info.value).__name__ == g["error"]
        assert str(info.value).replace(str(p), "<path>") == g["message"]
    else:
        m = lc.load_model(p, format=g["format"])
        assert (lc.model_digest(m), m.xi, m.num_loops) == (g["digest"], g["xi"], g["num_loops"])
        assert model_io.recompute_xi(m) == m.xi


def test_unknown_format(tmp_path):
    with pytest.raises(model_io.ParseError, match="unknown model format"):
        lc.load_model(tmp_path / "x", format="obj")
