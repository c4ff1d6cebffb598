"""C5 accuracy/throughput sweep (BASELINE configs[4]) on the GPU, next to the
reference's CPU numbers from tests/golden/golden_c5.json.

    python tools/c5_sweep.py [--out profiles/r02/c5_table.md]

For ribbon (double_helix_ribbon(10, n), lambda = 10) and yarn (two adjacent
knit courses, W = 100, lambda = -100) at n = 1e3 .. 1e6 segments per loop:
GPU direct summation in the three arithmetic forms (kernel time by CUDA
events, |raw - lambda|), the GPU Barnes-Hut forest (build + traversal), and
the reference's DS / BH / CC times and errors (one core, this build
container; DS at 1e6 extrapolated by n^2 from 1e5).
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import c5_cases  # noqa: E402
import paper_2106_12655_b200 as lc  # noqa: E402
from paper_2106_12655_b200 import _native  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    g = c5_cases.golden()
    ctx = _native.context()
    modes = [("phase", _native.GAUSS_PHASE), ("atan", _native.GAUSS_ATAN), ("ref", _native.GAUSS_REF),
             ("anglesum", _native.GAUSS_ANGLESUM)]
    rows = []
    hdr = ("| case | n | seg-pairs | GPU DS phase ms | err | GPU DS atan ms | err | GPU DS ref ms | err | "
           "GPU DS anglesum ms | err | GPU BH ms (build+eval) | BH err | ref DS s | ref DS err | ref BH s | "
           "ref BH err | ref CC s | ref CC |")
    rows.append(hdr)
    rows.append("|" + "|".join(["---"] * (hdr.count("|") - 1)) + "|")
    for name in c5_cases.NAMES:
        for n in c5_cases.NS:
            rec = g[f"{name}/{n}"]
            (a, b), lam = c5_cases.loops(name, n)
            assert [c5_cases.sha(a), c5_cases.sha(b)] == rec["sha256"]
            cells = [name, f"{n:.0e}", f"{float(n) * n:.1e}"]
            for label, mode in modes:
                if label in ("ref", "anglesum") and n > 100_000:
                    cells += ["—", "—"]
                    continue
                ctx.link_direct(a, b, mode)                      # warm
                raw = ctx.link_direct(a, b, mode)
                ms = ctx.last_gauss_ms()
                cells += [f"{ms:.3f}", f"{abs(raw - lam):.1e}"]
                print(f"{name}/{n} {label}: raw {raw!r} kernel {ms:.3f} ms", flush=True)
            pa, pb = lc.PolylineLoop(a), lc.PolylineLoop(b)
            lc.barnes_hut_detailed(lc.build_moment_tree(pa), lc.build_moment_tree(pb))
            t0 = time.perf_counter()
            ta, tb = lc.build_moment_tree(pa), lc.build_moment_tree(pb)
            t1 = time.perf_counter()
            bh = lc.barnes_hut_detailed(ta, tb)
            t2 = time.perf_counter()
            cells += [f"{1e3 * (t1 - t0):.2f}+{1e3 * (t2 - t1):.2f}", f"{abs(bh.value - lam):.1e}"]
            if "ds_raw" in rec:
                cells += [f"{rec['ds_seconds']:.2f}", f"{abs(rec['ds_raw'] - lam):.1e}"]
            else:
                cells += [f"~{rec['ds_seconds_extrapolated']:.0f} (extrap.)", "—"]
            cells += [f"{rec['bh_build_seconds'] + rec['bh_eval_seconds']:.3f}", f"{abs(rec['bh_value'] - lam):.1e}",
                      f"{rec['cc_seconds']:.3f}", str(rec.get("cc_value", rec.get("cc_error")))]
            rows.append("| " + " | ".join(cells) + " |")
    text = "\n".join(rows)
    print(text)
    if args.out:
        Path(args.out).write_text(
            "# C5 accuracy/throughput sweep (B200 GPU vs the reference on one CPU core)\n\n"
            "GPU: tools/c5_sweep.py (kernel times by CUDA events; BH = GPU moment forest build + traversal, "
            "wall time). Reference: tests/golden/golden_c5.json (tests/golden/make_golden_c5.py, the reference "
            "package run in the build container, one core). err = |value - exact lambda|.\n\n" + text + "\n")


if __name__ == "__main__":
    main()
