"""cProfile of one verify() on the Kusari tube (GPU box): where the host time goes."""
import cProfile, os, pstats, sys, time, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2106_12655_b200 as lc
from paper_2106_12655_b200 import generators as gen
before, after = gen.kusari_tube(), gen.kusari_tube(after=True)
cert = lc.compute_linking_matrix(before)
warnings.simplefilter("ignore")
for _ in range(5):
    lc.verify(after, cert)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); lc.verify(after, cert); ts.append(1e3 * (time.perf_counter() - t0))
print("verify ms", [round(t, 2) for t in ts])
pr = cProfile.Profile()
pr.enable()
lc.verify(after, cert)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
