"""C4 parity slice ("full DS parity on a 10k-segment version"):
the interlocking-course knit tube with 10,000-segment courses, run through
the REFERENCE's compute_linking_matrix and link_direct (this container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_c4.py

Writes tests/golden/golden_c4.json (certificate, raw value per PLS pair,
model fingerprint).
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import linkcert as ref  # noqa: E402

import cases  # noqa: E402
from make_golden import to_ref  # noqa: E402
from paper_2106_12655_b200 import generators as ours  # noqa: E402

COURSES, N, W = 5, 10_000, 100


def main():
    model = ours.knit_tube(courses=COURSES, n=N, W=W)
    rm = to_ref(model)
    t0 = time.perf_counter()
    mat = ref.compute_linking_matrix(rm)
    t1 = time.perf_counter()
    pairs = list(ref.potential_link_search(rm))
    polys = ref.discretize(rm, ref.potential_link_search(rm))
    raw = {f"{i},{j}": ref.link_direct(polys[i], polys[j]) for i, j in pairs}
    out = {"courses": COURSES, "n": N, "W": W, "fingerprint": cases.fingerprint(model),
           "entries": [list(e) for e in mat.entries], "digest": mat.model_digest, "raw": raw,
           "vertices_per_loop": [len(p) for p in polys], "reference_seconds": t1 - t0}
    (HERE / "golden_c4.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    print(json.dumps({k: out[k] for k in ("entries", "raw", "reference_seconds")}))


if __name__ == "__main__":
    main()
