"""Per-kernel table of the last device step in an ncu launch list (--metrics gpu__time_duration.sum CSV).

usage: python tools/step_table.py launches.csv [first_kernel_regex]
The step is taken as the kernels from the last occurrence of the first-kernel
pattern (default: seg_boxes) to the end of the list.
"""
import collections
import csv
import re
import sys

path = sys.argv[1]
first = re.compile(sys.argv[2] if len(sys.argv) > 2 else "seg_boxes")
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
starts = [i for i, (k, _) in enumerate(recs) if first.search(k)]
start = starts[-1]            # the last step in the list runs to its end
step = [r for r in recs[start:] if "dfma_chain" not in r[0]]   # not the bench's peak probe
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
