"""Overlap summary of an SN_TIMELINE launch timeline (sn_abi.cu; CUDA events per launch).

  python tools/timeline_summary.py timeline.csv

Columns: kind (0 window, 1 left, 2 right, 3 Q, 4 scan), level, stream (0 critical path, 1
remaining strips, 2 Q), start_ms, end_ms.  Event intervals include queueing behind other
work on the same stream only (stream order), so busy time per stream is the union of its
intervals.  Reports per stream busy time, per kind time, and how much of the window-kernel
(critical path) time runs concurrently with panel work on the other streams -- the W/L/R/Q
overlap of the level executor."""
import csv
import json
import sys


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def length(iv):
    return sum(b - a for a, b in iv)


def intersect(x, y):
    i = j = 0
    out = []
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if a < b:
            out.append([a, b])
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return out


rows = [r for r in csv.DictReader(open(sys.argv[1]))]
recs = [(int(r["kind"]), int(r["level"]), int(r["stream"]), float(r["start_ms"]), float(r["end_ms"])) for r in rows]
recs = [r for r in recs if r[3] >= 0]
span = max(r[4] for r in recs) - min(r[3] for r in recs)
names = {0: "window", 1: "left", 2: "right", 3: "q", 4: "scan"}
by_stream = {s: union([[a, b] for k, l, st, a, b in recs if st == s]) for s in (0, 1, 2)}
by_kind = {names[k]: union([[a, b] for kk, l, st, a, b in recs if kk == k]) for k in names}
win = by_kind["window"]
other = union(by_stream[1] + by_stream[2])
crit_panels = union([[a, b] for k, l, st, a, b in recs if st == 0 and k in (1, 2)])
out = {
    "span_ms": span,
    "levels": 1 + max(r[1] for r in recs),
    "busy_ms": {"critical_stream": length(by_stream[0]), "rest_stream": length(by_stream[1]),
                "q_stream": length(by_stream[2])},
    "kind_ms": {k: length(v) for k, v in by_kind.items()},
    "window_ms": length(win),
    "window_overlapped_by_rest_or_q_ms": length(intersect(win, other)),
    "window_overlap_fraction": length(intersect(win, other)) / max(1e-9, length(win)),
    "critical_panels_overlapped_by_q_ms": length(intersect(crit_panels, by_stream[2])),
    "any_two_streams_busy_ms": length(union(intersect(by_stream[0], by_stream[1]) + intersect(by_stream[0], by_stream[2])
                                            + intersect(by_stream[1], by_stream[2]))),
}
print(json.dumps(out, indent=1))
