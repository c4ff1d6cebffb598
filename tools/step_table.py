"""Per-kernel table of the last device step in an ncu launch list (--metrics gpu__time_duration.sum CSV).

usage: python tools/step_table.py launches.csv [first_kernel_regex]
A step is the run of kernels from one occurrence of the first-kernel pattern
(default: loop_grid_kernel, the fused graph's first kernel) to the next; the table
shows the last step that ran the fused pair Gauss kernel (bench.py's timed
steps), not the e2e verifies, the standalone kernel timing or the peak probes
that follow them in the list.
"""
import collections
import csv
import re
import sys

path = sys.argv[1]
first = re.compile(sys.argv[2] if len(sys.argv) > 2 else "loop_grid_kernel|prezero_kernel")
rows = list(csv.reader(open(path)))
hdr, recs = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = re.sub(r"\(.*", "", d["Kernel Name"])[:80]
        recs.append((name, float(d["Metric Value"].replace(",", "")) / 1000.0))
starts = [i for i, (k, _) in enumerate(recs) if first.search(k)] + [len(recs)]
steps = [recs[a:b] for a, b in zip(starts, starts[1:])]
probe = re.compile("dfma_chain|dmma_chain|gauss_items_kernel|item_pair|pair_geom_kernel")
steps = [[r for r in st if not probe.search(r[0])] for st in steps if any("gauss_pairs" in k for k, _ in st)]
step = steps[-1]
tot = sum(v for _, v in step)
agg = collections.OrderedDict()
for k, v in step:
    a = agg.setdefault(k, [0.0, 0])
    a[0] += v
    a[1] += 1
print("| kernel | launches | us | share |")
print("|---|---|---|---|")
for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"| `{k}` | {n} | {v:.1f} | {100 * v / tot:.1f}% |")
print(f"| **sum ({len(step)} launches)** | | **{tot:.1f}** | |")
