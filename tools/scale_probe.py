"""Larger-than-benchmark models through the fused path (GPU box): correctness vs the
oracle on the integers and the device time per certificate."""
import os, sys, time, warnings
os.environ.setdefault("LINKCERT_STAGE_TIMES", "1")   # every stage timed (diagnostic)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native, generators as gen
from paper_2106_12655_b200.certify import device_step, excluded_keys
from paper_2106_12655_b200.pls import upload
import linkcert_oracle as orc
for rows in (98, 196):
    m = gen.kusari_tube(n_around=95, rows=rows, partial=81)
    ctx = _native.context()
    upload(m, ctx)
    prm = lc.DiscretizationParams()
    for _ in range(4):
        pairs, raw, lk, flags = device_step(ctx, m.xi, excluded_keys(()), prm)
    st = ctx.stage_times()
    c, t, o = m.packed()
    t0 = time.time()
    want_pairs = orc.pls(c, t, o)
    ok_pairs = np.array_equal(np.asarray(pairs), want_pairs)
    nv = np.diff(o)
    sp = int(np.sum(nv[want_pairs[:, 0]] * nv[want_pairs[:, 1]]))
    print(f"rows {rows}: loops {m.num_loops} pairs {len(pairs)} pairs==oracle {ok_pairs} links {int(np.sum(lk != 0))} "
          f"path {ctx.last_run_fused()} device {st['begin_to_reduce']:.3f} ms -> {sp / st['begin_to_reduce'] / 1e-3:.3e} "
          f"seg-pairs/s", flush=True)
