"""Where the step time outside the library's begin -> reduce events goes (GPU box):
host time of the C-ABI call, and the event-timed step with the GPU idle at launch
(as bench.py) vs busy (a torch sleep kernel queued first hides the host launch).
    python tools/launch_probe.py
"""
import os
os.environ.setdefault("LINKCERT_STAGE_TIMES", "1")   # every stage timed (diagnostic)
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2106_12655_b200 import _native, generators as gen  # noqa: E402
from paper_2106_12655_b200.certify import device_step, excluded_keys  # noqa: E402
from paper_2106_12655_b200.discretize import DiscretizationParams  # noqa: E402
from paper_2106_12655_b200.pls import upload  # noqa: E402


def main():
    torch.cuda.set_device(0)
    m = gen.kusari_tube(after=True)
    ctx = _native.context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    upload(m, ctx)
    ex, prm = excluded_keys(()), DiscretizationParams()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    # sleep kernel duration
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); torch.cuda._sleep(200_000); e1.record(stream); torch.cuda.synchronize()
    sleep_ms = e0.elapsed_time(e1)
    for busy in (False, True, False, True):
        ms, host_ms, call_ms, b2r = [], [], [], []
        for k in range(35):
            flush.zero_()
            torch.cuda.synchronize()
            e0.record(stream)
            if busy:
                torch.cuda._sleep(200_000)
            t0 = time.perf_counter()
            device_step(ctx, m.xi, ex, prm)
            t1 = time.perf_counter()
            e1.record(stream)
            torch.cuda.synchronize()
            if k >= 5:
                ms.append(e0.elapsed_time(e1) - (sleep_ms if busy else 0.0))
                host_ms.append(1e3 * (t1 - t0))
                b2r.append(ctx.stage_times()["begin_to_reduce"])
        print(f"{'busy' if busy else 'idle'}: step {statistics.median(ms):.4f} ms  begin_to_reduce "
              f"{statistics.median(b2r):.4f}  device_step host {statistics.median(host_ms):.4f} ms "
              f"(sleep {sleep_ms:.3f} ms)", flush=True)
    # host cost of the call alone: the run_pipeline C-ABI call split from the python around it
    args = (ex, m.xi, prm.epsilon, prm.max_passes, prm.max_subsegments, _native.GAUSS_PHASE)
    ts = []
    for k in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.run_pipeline(*args)
        ts.append(1e3 * (time.perf_counter() - t0))
    print(f"run_pipeline host (incl. its sync): {statistics.median(ts[5:]):.4f} ms")


if __name__ == "__main__":
    main()
