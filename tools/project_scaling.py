"""Projection of the sharded reordering's P-GPU time from a one-GPU launch list (VERDICT r1
item 4: a measured projection, not an estimate).

  python tools/project_scaling.py launches.csv [levels]

Input: an ncu --metrics gpu__time_duration.sum launch list of one bench step (config 3, the
bench launch configuration: per level window kernel, critical left/right strips, remaining
left/right strips, Q update).  Every launch's duration is measured alone (ncu serialises), so
they are the isolated per-level component times.  Model of the sharded executor
at P ranks, per level l:
  critical path  W_l + crit_l + comm_l          (the window tasks of a level run concurrently
                                                 on their owners; the critical strips on the
                                                 owners of the next level's windows; comm_l =
                                                 the level's Z broadcast + straddle pulls/pushes)
  throughput     (crit_l + rest_l + Q_l) / P    (the panels split evenly: S column blocks are
                                                 block-cyclic, Q rows contiguous)
  T(P) = sum_l max(critical path, throughput)   (the remaining strips and Q overlap the next
                                                 level's window tasks, as on one GPU)
comm_l = 25 us latency per NCCL group + the level's Z bytes (k x 256 x 8 per window) / 300 GB/s.
The one-GPU row uses the same model with P = 1 and comm = 0 and is compared with the measured
step to calibrate it."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Grid Size")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
seq = []
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki]
    kind = "W" if "window_kernel" in name else ("L" if "<256, 0>" in name else ("R" if "<256, 1>" in name else ("Q" if "<256, 2>" in name else "?")))
    grid = int(r[gi].strip("()").split(",")[0])
    seq.append((kind, float(r[vi].replace(",", "")) * scale[r[ui]], grid))
# split into levels (each starts with a window kernel); keep the last step's levels
levels = []
for k, t, g in seq:
    if k == "W":
        levels.append({"W": t, "nwin": g, "parts": []})
    elif levels:
        levels[-1]["parts"].append((k, t))
nlev = int(sys.argv[2]) if len(sys.argv) > 2 else 203
# the lookahead step's levels (5 launches after the window kernel: L crit, R crit, L rest,
# R rest, Q); the bench's extra isolated step (lookahead off: L, R, Q) is skipped
levels = [lv for lv in levels if len(lv["parts"]) == 5][-nlev:]
tot = collections.Counter()
model = {}
for lv in levels:
    parts = lv["parts"]
    # launch order per level: L crit, R crit, L rest, R rest, Q
    crit = sum(t for k, t in parts[:2])
    rest = sum(t for k, t in parts[2:4])
    q = sum(t for k, t in parts if k == "Q")
    lv.update(crit=crit, rest=rest, q=q)
    tot["W"] += lv["W"]; tot["crit"] += crit; tot["rest"] += rest; tot["Q"] += q
for P in (1, 2, 4, 8):
    T = 0.0
    for lv in levels:
        comm = 0.0 if P == 1 else 0.025 + lv["nwin"] * 256 * 256 * 8 / 300e9 * 1e3
        T += max(lv["W"] + lv["crit"] + comm, (lv["crit"] + lv["rest"] + lv["q"]) / P)
    model[P] = T
out = {"levels": len(levels), "component_ms": dict(tot),
       "window_chain_ms": tot["W"], "projected_ms": model,
       "projected_speedup": {P: model[1] / model[P] for P in model}}
print(json.dumps(out, indent=1))
