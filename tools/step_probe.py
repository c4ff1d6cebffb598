"""Stage times of the fused device step under different conditions (GPU box; not a bench number).
    python tools/step_probe.py [--flush] [--serial-checks]"""
import argparse, os, statistics, sys
os.environ.setdefault("LINKCERT_STAGE_TIMES", "1")   # every stage timed (diagnostic)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--flush", action="store_true")
a = ap.parse_args()
import torch
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native, generators as gen
from paper_2106_12655_b200.certify import device_step, excluded_keys
from paper_2106_12655_b200.pls import upload
m = gen.kusari_tube(after=True)
ctx = _native.context()
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
upload(m, ctx)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = []
for k in range(40):
    if a.flush:
        flush.zero_()
    torch.cuda.synchronize()
    device_step(ctx, m.xi, excluded_keys(()), lc.DiscretizationParams())
    if k >= 10:
        st.append(ctx.stage_times())
print({key: round(statistics.mean(s[key] for s in st), 4) for key in st[0]}, "flush" if a.flush else "no flush",
      os.environ.get("LINKCERT_EXP_SERIAL_CHECKS", ""))
