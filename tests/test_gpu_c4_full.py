"""C4 at full scale (BASELINE configs[3]): 200 knit courses x 100,000 segments,
1.99e12 segment pairs, against the reference (tests/golden/golden_c4_full.json,
made by tests/golden/make_golden_c4_full.py in the build container):

* the model is rebuilt bitwise (per-course sha256 of the reference's input);
* PLS pairs == the reference's potential_link_search (199 adjacent pairs);
* every integer == the reference's crossing count (link_count_crossings);
* raw sums of the sampled pairs within 1e-9 of the reference's link_direct
  (1e10 segment pairs each, ~540 s per pair on one reference core).
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2106_12655_b200 as lc
from paper_2106_12655_b200.certify import run_device_pipeline

pytestmark = pytest.mark.gpu

G = json.loads((Path(__file__).resolve().parent / "golden" / "golden_c4_full.json").read_text())


def test_c4_full_scale_vs_reference(gpu):
    model = lc.generators.knit_tube(courses=G["courses"], n=G["n"], W=G["W"])
    hashes = [hashlib.sha256(np.ascontiguousarray(lp.control_points).tobytes()).hexdigest() for lp in model.loops]
    assert hashes == G["course_sha256"]
    pairs, raw, lk, flags, _ = run_device_pipeline(model)
    pairs, raw, lk, flags = pairs.copy(), raw.copy(), lk.copy(), flags.copy()
    assert pairs.tolist() == G["pls_pairs"]
    assert not flags.any()
    cc = np.array([G["cc"][f"{i},{j}"] for i, j in pairs.tolist()])
    assert np.array_equal(lk, cc)
    pos = {(int(i), int(j)): k for k, (i, j) in enumerate(pairs.tolist())}
    for key, want in G["ds_raw"].items():
        i, j = map(int, key.split(","))
        assert abs(raw[pos[(i, j)]] - want) < 1e-9, (key, raw[pos[(i, j)]], want)
    mat = lc.compute_linking_matrix(model)
    assert mat.entries == tuple((k, k + 1, -G["W"]) for k in range(G["courses"] - 1))
