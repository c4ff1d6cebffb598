"""Median stage times of the fused Kusari step (CUDA events of the library), with or
without an L2 flush between steps — for A/B builds (LINKCERT_LIB=...).  GPU box:
    python tools/stage_ab.py [--flush] [--steps 30]
"""
import argparse
import os
os.environ.setdefault("LINKCERT_STAGE_TIMES", "1")   # every stage timed (diagnostic)
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2106_12655_b200 import _native, generators as gen  # noqa: E402
from paper_2106_12655_b200.certify import device_step, excluded_keys  # noqa: E402
from paper_2106_12655_b200.discretize import DiscretizationParams  # noqa: E402
from paper_2106_12655_b200.pls import upload  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--flush", action="store_true")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--label", default="")
    ap.add_argument("--torch-stream", action="store_true", help="run on torch's current stream (as bench.py)")
    ap.add_argument("--bench-model", action="store_true", help="bench.py's model (from_polyline_arrays)")
    ap.add_argument("--torch-first", action="store_true", help="torch.cuda.set_device before the library (as bench.py)")
    ap.add_argument("--getpoly", action="store_true", help="ctx.get_polylines() after the first step (as bench.py)")
    ap.add_argument("--flush-first", action="store_true", help="allocate the flush buffer before the upload")
    ap.add_argument("--cert", action="store_true", help="compute the 'before' certificate first (as bench.py)")
    a = ap.parse_args()
    import torch
    if a.torch_first:
        torch.cuda.set_device(0)
        torch.empty(1, device="cuda")
    if a.bench_model:
        import bench
        from paper_2106_12655_b200.geometry import CurveModel
        m = CurveModel.from_polyline_arrays(*bench.workload_arrays("kusari")[1])
    else:
        m = gen.kusari_tube(after=True)
    ctx = _native.context(0)
    if a.torch_stream:
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    if a.flush_first:
        flush0 = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    if a.cert:
        import paper_2106_12655_b200 as lc
        lc.compute_linking_matrix(gen.kusari_tube())
    upload(m, ctx)
    flush = (flush0 if a.flush_first else torch.empty(512 << 20, dtype=torch.uint8, device="cuda")) if a.flush else None
    rows = []
    for i in range(a.steps + 5):
        if flush is not None:
            flush.zero_()
            torch.cuda.synchronize()
        device_step(ctx, m.xi, excluded_keys(()), DiscretizationParams())
        if i == 0 and a.getpoly:
            ctx.get_polylines()
        if i >= 5:
            rows.append(ctx.stage_times())
    med = {k: round(float(np.median([r[k] for r in rows])), 4) for k in rows[0]}
    print(a.label, "flush" if a.flush else "hot", "torch-stream" if a.torch_stream else "",
          "bench-model" if a.bench_model else "", "cert" if a.cert else "", "torch-first" if a.torch_first else "", "getpoly" if a.getpoly else "", "flush-first" if a.flush_first else "", med, flush=True)


if __name__ == "__main__":
    main()
