"""CPU-only checks of the C-ABI library: it loads, exports every declared symbol,
its ctypes table matches the header, and it refuses to compute without a GPU."""

import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2106_12655_b200 import _native, build

HEADER = ROOT / "include" / "linkcert_b200.h"


def header_symbols():
    text = HEADER.read_text()
    return set(re.findall(r"LC_API\s+[\w\s\*]+?\b(lc_\w+)\s*\(", text))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _native.load_library()


def test_library_exports_every_header_symbol(lib):
    import subprocess

    syms = header_symbols()
    assert len(syms) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\sT\s(lc_\w+)", out))
    assert syms <= exported, sorted(syms - exported)
    for s in syms:
        assert hasattr(lib, s)


def test_ctypes_table_matches_header():
    assert set(_native.SIGNATURES) == header_symbols()


def test_abi_version(lib):
    assert lib.lc_abi_version() == 2


def test_no_device_means_loud_failure():
    """No CUDA device here: the product path raises instead of computing on the CPU."""
    count = np.zeros(1, dtype=np.int32)
    rc = _native.load_library().lc_device_count(count.ctypes.data_as(_native.ctypes.POINTER(_native.ctypes.c_int)))
    if rc == _native.LC_OK and count[0] > 0:
        pytest.skip("a CUDA device is visible")
    import paper_2106_12655_b200 as lc

    _native._ctx.clear()
    with pytest.raises(_native.NativeUnavailable):
        lc.link_direct(np.eye(3), np.eye(3) + 5.0)
    with pytest.raises(_native.NativeUnavailable):
        lc.compute_linking_matrix(lc.generators.hopf(16)[0])


def test_missing_library_is_loud(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "LIB_PATH", tmp_path / "missing.so")
    monkeypatch.setattr(_native, "_lib", None)
    with pytest.raises(_native.NativeUnavailable):
        _native.load_library()


def test_float_repr_matches_cpython(lib):
    rng = np.random.default_rng(3)
    xs = list(rng.normal(size=4000) * 10.0 ** rng.integers(-40, 40, size=4000)) + list(rng.random(1000))
    xs += [0.0, -0.0, 1.0, -1.0, 1e16, 1e15, 9.999999999999999e15, 1e-5, 1e-4, 5e-324, 1.7976931348623157e308,
           0.1, 1 / 3, 123456789012345678.0, 2.5, 1e22, -1e-7]
    xs += [10.0 ** k for k in range(-320, 309)] + [float(k) for k in range(-1000, 1000, 7)]
    bad = [x for x in xs if _native.float_repr(x) != repr(float(x))]
    assert not bad, bad[:5]


def test_float_repr_bulk_fuzz(lib):
    """Dragonbox digest formatter vs CPython repr over all double classes (and
    the std::to_chars cross-check formatter on the same values)."""
    rng = np.random.default_rng(11)
    n = 40000
    xs = np.concatenate([
        rng.integers(0, 0x7FF0000000000000, n, dtype=np.int64).view(np.float64),      # any finite bit pattern
        np.ldexp(1.0, rng.integers(-1074, 1024, n)),                                   # shorter-interval case
        np.ldexp(1.0 + rng.integers(0, 4, n) * 2.0 ** -52, rng.integers(-1074, 1023, n)),
        rng.integers(-2 ** 62, 2 ** 62, n).astype(np.float64),
        rng.integers(1, 1 << 52, n, dtype=np.int64).view(np.float64),                 # subnormals
        np.round(rng.random(n) * 10.0 ** rng.integers(0, 17, n)) / 10.0 ** rng.integers(0, 20, n),
    ])
    xs *= np.where(rng.random(len(xs)) < 0.5, -1.0, 1.0)
    truth = [repr(x) for x in xs.tolist()]
    assert _native.float_repr_many(xs) == truth
    assert _native.float_repr_many(xs, use_tochars=True) == truth


@pytest.mark.parametrize("n", [0, 1, 55, 56, 57, 63, 64, 65, 119, 120, 128, 1000, 100003])
def test_sha256_both_paths(lib, n):
    import hashlib

    data = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8).tobytes()
    fast, _ = _native.sha256_hex(data)
    portable, _ = _native.sha256_hex(data, force_portable=True)
    assert fast == portable == hashlib.sha256(data).hexdigest()
