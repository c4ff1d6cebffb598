"""C5 (BASELINE configs[4]): FP64 direct summation at 1e3..1e6 segments per loop
against the reference's own direct sum, Barnes-Hut and crossing count
(tests/golden/golden_c5.json, made by tests/golden/make_golden_c5.py).

* integers: round(raw) == the known lambda == the reference's crossing count;
* raw: within 1e-9 of the reference's DS raw (n <= 1e5, where the reference
  ran: 1e10 segment pairs took it ~520 s) and of the exact lambda at n = 1e6
  (1e12 segment pairs; the reference's DS would need ~14 h);
* Barnes-Hut (the GPU forest, default BarnesHutParams): value within 1e-9 of
  the reference's, same adaptive decision and beta.
The accuracy/time table is tools/c5_sweep.py -> profiles/r02/c5_table.md.
"""

import pytest

import c5_cases
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native

pytestmark = pytest.mark.gpu

RAW_TOL = 1e-9
G = c5_cases.golden()


@pytest.mark.parametrize("n", c5_cases.NS)
@pytest.mark.parametrize("name", c5_cases.NAMES)
def test_c5_direct_sum(gpu, name, n):
    g = G[f"{name}/{n}"]
    (a, b), lam = c5_cases.loops(name, n)
    assert [c5_cases.sha(a), c5_cases.sha(b)] == g["sha256"]
    modes = [_native.GAUSS_PHASE, _native.GAUSS_ATAN] + ([_native.GAUSS_REF] if n <= 100_000 else [])
    for mode in modes:
        raw = gpu.link_direct(a, b, mode)
        assert round(raw) == lam == g["cc_value"]
        assert abs(raw - lam) < RAW_TOL, (mode, raw)
        if "ds_raw" in g:
            assert abs(raw - g["ds_raw"]) < RAW_TOL, (mode, raw, g["ds_raw"])


@pytest.mark.parametrize("n", c5_cases.NS)
@pytest.mark.parametrize("name", c5_cases.NAMES)
def test_c5_barnes_hut_vs_reference(gpu, name, n):
    g = G[f"{name}/{n}"]
    (a, b), _ = c5_cases.loops(name, n)
    res = lc.barnes_hut_detailed(lc.build_moment_tree(lc.PolylineLoop(a)), lc.build_moment_tree(lc.PolylineLoop(b)))
    assert res.reran == g["bh_reran"]
    assert res.beta_used == pytest.approx(g["bh_beta_used"], rel=1e-12)
    assert abs(res.value - g["bh_value"]) < RAW_TOL
