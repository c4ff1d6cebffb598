"""C5 sweep inputs (BASELINE configs[4]) rebuilt on the box: the same vertex
arrays tests/golden/make_golden_c5.py handed the reference (sha256-checked)."""

import hashlib
import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden_c5.json"
NS = (1_000, 10_000, 100_000, 1_000_000)
NAMES = ("ribbon", "yarn")


def golden():
    return json.loads(GOLDEN.read_text())


def loops(name, n):
    """(a, b) vertex arrays of case name/n and its exact linking number."""
    from paper_2106_12655_b200 import generators as gen

    if name == "ribbon":
        m, _ = gen.double_helix_ribbon(10, n)
        return [np.ascontiguousarray(lp.control_points) for lp in m.loops], 10
    return [gen.knit_course(0, n), gen.knit_course(1, n)], -100


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
