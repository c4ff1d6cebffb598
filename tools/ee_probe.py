"""Device early exit on the Kusari tube (GPU box): report, pairs evaluated, times."""
import os, sys, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import _native, generators as gen
warnings.simplefilter("ignore")
before, after = gen.kusari_tube(), gen.kusari_tube(after=True)
cert = lc.compute_linking_matrix(before)
ctx = _native.context()
for k in range(4):
    t0 = time.perf_counter()
    rep = lc.verify(after, cert, early_exit=True)
    t1 = time.perf_counter()
    print(f"early exit: {rep.status} first={rep.first_failure} destroyed={rep.destroyed} "
          f"stats(place, evaluated)={ctx.early_exit_stats()} {1e3 * (t1 - t0):.1f} ms", flush=True)
t0 = time.perf_counter()
full = lc.verify(after, cert)
print(f"full verify: {full.status} {1e3 * (time.perf_counter() - t0):.1f} ms, P={len(lc.potential_link_search(after))}")
for k in range(2):
    t0 = time.perf_counter()
    mb = lc.compute_linking_matrix(before, choice=lc.KernelChoice(method="bh"))
    print(f"bh certificate: {len(mb.entries)} entries equal DS={mb.entries == cert.entries} "
          f"{1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
