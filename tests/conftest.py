"""Shared test fixtures.  `-m gpu` tests need a B200 and the built library."""

import json
import math
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and liblinkcert_b200.so")
    # the library (and the oracle) are built in-tree by __graft_entry__.build();
    # build them here only if they are missing (nvcc cross-compiles without a GPU)
    from paper_2106_12655_b200 import build

    if not build.LIB.exists():
        build.build()
    if not (ROOT / "oracle" / "liboracle_gauss.so").exists():
        import linkcert_oracle

        linkcert_oracle.build()


def circle_points(n, center=(0.0, 0.0, 0.0), u=(1.0, 0.0, 0.0), v=(0.0, 1.0, 0.0), radius=1.0):
    """Ring vertices in the reference test helper's expression order (conftest.py:11-17)."""
    t = np.linspace(0.0, 2.0 * math.pi, n, endpoint=False)
    return (np.asarray(center, dtype=float) + radius * np.outer(np.cos(t), np.asarray(u, dtype=float))
            + radius * np.outer(np.sin(t), np.asarray(v, dtype=float)))


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN / "golden.json") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_arrays():
    with np.load(GOLDEN / "golden_arrays.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def oracle():
    import linkcert_oracle

    linkcert_oracle.lib()
    return linkcert_oracle


def _cuda_ok():
    try:
        from paper_2106_12655_b200 import _native

        _native.context()
        return True
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    """The native context; GPU tests fail loudly (no silent CPU path) if it cannot be created."""
    from paper_2106_12655_b200 import _native

    return _native.context()


@pytest.fixture(scope="session")
def bh_golden():
    with open(GOLDEN / "bh_golden.json") as f:
        return json.load(f)


@pytest.fixture(scope="session")
def bh_arrays():
    with np.load(GOLDEN / "bh_golden.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def bh_oracle():
    import bh_oracle

    return bh_oracle
