"""C4 parity slice: the interlocking-course knit tube with
10,000-segment courses (4 PLS pairs x 1e8 segment pairs), against the
reference's own certificate and raw link values (tests/golden/golden_c4.json,
make_golden_c4.py; the reference took ~21 s).

CPU: the oracle reproduces the raw sums BITWISE.  GPU: the CUDA path gives
the same certificate and raw sums within 1e-9.
"""

import json
from pathlib import Path

import numpy as np
import pytest

import cases
import paper_2106_12655_b200 as lc

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_c4.json"


@pytest.fixture(scope="module")
def c4():
    g = json.loads(GOLDEN.read_text())
    model = lc.generators.knit_tube(courses=g["courses"], n=g["n"], W=g["W"])
    assert cases.fingerprint(model) == g["fingerprint"]
    return g, model


def test_c4_slice_oracle_bitwise(oracle, c4):
    g, model = c4
    coeffs, t, off = model.packed()
    pairs = oracle.pls(coeffs, t, off)
    assert [f"{i},{j}" for i, j in pairs.tolist()] == sorted(g["raw"], key=lambda k: tuple(map(int, k.split(","))))
    verts, voff = oracle.discretize(coeffs, t, off, model.xi, pairs)
    assert np.diff(voff).tolist() == g["vertices_per_loop"]
    raw = oracle.evaluate_pairs(verts, voff, pairs)
    assert [float(r) for r in raw] == [g["raw"][f"{i},{j}"] for i, j in pairs.tolist()]


@pytest.mark.gpu
def test_c4_slice_gpu(gpu, c4):
    from paper_2106_12655_b200.certify import run_device_pipeline

    g, model = c4
    mat = lc.compute_linking_matrix(model)
    assert [list(e) for e in mat.entries] == g["entries"]
    assert mat.model_digest == g["digest"]
    pairs, raw = (np.array(a).copy() for a in run_device_pipeline(model)[:2])
    assert [f"{i},{j}" for i, j in pairs.tolist()] == list(sorted(g["raw"], key=lambda k: tuple(map(int, k.split(",")))))
    for (i, j), r in zip(pairs.tolist(), raw.tolist()):
        assert abs(r - g["raw"][f"{i},{j}"]) <= 1e-9
