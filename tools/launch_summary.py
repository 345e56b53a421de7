"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
gi = h.index("Grid Size")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    key = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "").replace("(anonymous namespace)::", "")
    agg[key][0] += 1
    agg[key][1] += float(r[vi].replace(",", "")) * scale[r[ui]]
tot = sum(a[1] for a in agg.values())
print("ncu --metrics gpu__time_duration.sum --clock-control none (cold cache, serialised)")
if len(sys.argv) > 2:
    print("command:", " ".join(sys.argv[2:]))
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-40s launches=%6d total=%10.1f ms share=%.3f avg=%.3f ms" % (k, c, t, t / tot, t / c))
