"""Device timeline of the fused step (debug marks, LINKCERT_TIMELINE=1): microseconds
from the first mark to the end of each stage, main stream and the two side branches
(S0: segment boxes + chords, S1: pass-1 checks).  GPU box:
    LINKCERT_TIMELINE=1 python tools/timeline.py [--workload kusari|e4in1] [--steps 6]
"""
import argparse
import os
os.environ.setdefault("LINKCERT_STAGE_TIMES", "1")   # every stage timed (diagnostic)
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("LINKCERT_TIMELINE", "1")

from paper_2106_12655_b200 import _native, generators as gen  # noqa: E402
from paper_2106_12655_b200.certify import device_step, excluded_keys  # noqa: E402
from paper_2106_12655_b200.discretize import DiscretizationParams  # noqa: E402
from paper_2106_12655_b200.pls import upload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="kusari", choices=["kusari", "e4in1"])
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--flush", action="store_true", help="write 512 MiB between steps (bench conditions)")
    a = ap.parse_args()
    m = gen.kusari_tube(after=True) if a.workload == "kusari" else gen.european_4in1(32, 32)
    ctx = _native.context(0)
    upload(m, ctx)
    flush = None
    if a.flush:
        import torch
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(a.steps):
        if flush is not None:
            flush.zero_()
            torch.cuda.synchronize()
        device_step(ctx, m.xi, excluded_keys(()), DiscretizationParams())
        print("stage ms", {k: round(v, 4) for k, v in ctx.stage_times().items()}, file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
