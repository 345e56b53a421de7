"""Hottest SASS lines of an ncu --page source --csv --print-source sass export, with the
sampled stall reasons: python tools/ncu_hot_sass.py source.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
h = rows[1]
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") or c.endswith("(samples)")]
data = []
for r in rows[2:]:
    if len(r) <= iall:
        continue
    try:
        v = int(r[iall])
    except ValueError:
        continue
    data.append((v, r))
tot = sum(v for v, _ in data) or 1
data.sort(key=lambda x: -x[0])
print("total samples", tot)
for v, r in data[:n]:
    print("%7d %5.1f%%  %-6s %s" % (v, 100.0 * v / tot, r[ia][-5:], r[isrc].strip()[:70]))
