"""Event-timed device step (as bench.py: L2 flushed, synchronized, e0 -> device_step -> e1),
median of N steps — for A/B of host-side launch costs (GPU box):
    [LINKCERT_STAGE_TIMES=1] python tools/step_time.py [--steps 60]"""
import argparse, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_12655_b200 import _native, generators as gen
from paper_2106_12655_b200.certify import device_step, excluded_keys
from paper_2106_12655_b200.discretize import DiscretizationParams
from paper_2106_12655_b200.pls import upload

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=60)
a = ap.parse_args()
m = gen.kusari_tube(after=True)
ctx = _native.context(0)
stream = torch.cuda.current_stream()
ctx.set_stream(stream.cuda_stream)
upload(m, ctx)
ex, prm = excluded_keys(()), DiscretizationParams()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for k in range(a.steps + 5):
    flush.zero_()
    torch.cuda.synchronize()
    e0.record(stream)
    device_step(ctx, m.xi, ex, prm)
    e1.record(stream)
    torch.cuda.synchronize()
    if k >= 5:
        ts.append(e0.elapsed_time(e1))
print(f"stage_times={os.environ.get('LINKCERT_STAGE_TIMES', '0')} step median {statistics.median(ts):.4f} ms "
      f"min {min(ts):.4f}", flush=True)
