"""Diagnosis of the config-2 pencil rejection: run the GPU path on windows
0..T-1 (schedule order), take window T's blocks of S and T back to the host, replay that
window's swaps with the oracle's swap in the GPU's step order, and for the first rejected swap
ask LAPACK dtgexc whether it would swap the same (n1+n2)^2 pencil block.

  python tools/pencil_rejection_probe.py [--config 2] [--window 1645]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402
from scipy.linalg import lapack  # noqa: E402

import oracle  # noqa: E402
import paper_1905_04975_b200 as sn  # noqa: E402
from workloads import CONFIGS, make_pencil  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--window", type=int, default=1645)
args = ap.parse_args()
c = CONFIGS[args.config]
p = make_pencil(c["n"], c["p2"], c["q"], c["sel"], c["psel"], c["w"], seed=1, device="cuda")
w = c["w"]
sub = (p.S.diagonal(1) != 0).cpu().numpy()
bmap = np.zeros(p.n, np.int8)
i = 0
while i < p.n - 1:
    if sub[i]:
        bmap[i], bmap[i + 1] = 1, 2
        i += 2
    else:
        i += 1
selrow = np.zeros(p.n, np.int8)
for r in range(p.n):
    selrow[r] = p.select[r]
for r in range(p.n - 1):
    if bmap[r] == 1:
        selrow[r] = selrow[r + 1] = 1 if (p.select[r] or p.select[r + 1]) else 0
sch = sn.schedule(bmap, selrow, w)
T = args.window
j1, k = int(sch["j1"][T]), int(sch["k"][T])
S, Tm = p.S.clone(), p.T.clone()
r = sn.reorder_pencil(S, Tm, None, None, p.select, window=w, max_windows=T)
torch.cuda.synchronize()
print("prefix run rc", r["rc"], "windows", r["stats"]["windows"])
D = np.asfortranarray(S.cpu().numpy().T[j1:j1 + k, j1:j1 + k])
E = np.asfortranarray(Tm.cpu().numpy().T[j1:j1 + k, j1:j1 + k])
sj, s1, s2 = sn.window_swaps(bmap, selrow, w, T)
last = -np.ones(k + 4, np.int64)
steps = []
for q in range(len(sj)):
    j = int(sj[q]) - j1
    m = int(s1[q]) + int(s2[q])
    t = max(last[j:j + m]) + 1
    last[j:j + m] = t
    steps.append(t)
order = sorted(range(len(sj)), key=lambda q: (steps[q], q))
L = oracle.lib()
ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
lapack_rejects = 0
for q in order:
    j = int(sj[q]) - j1
    n1, n2 = int(s1[q]), int(s2[q])
    m = n1 + n2
    A0, B0 = D[j:j + m, j:j + m].copy(order="F"), E[j:j + m, j:j + m].copy(order="F")
    if m == 4:
        info4 = lapack.dtgexc(A0.copy(), B0.copy(), np.eye(m), np.eye(m), n1 + 1, 1)[5]
        lapack_rejects += int(info4 != 0)
    if L.or_gswap(k, ptr(D), k, ptr(E), k, j, n1, n2, None, 0, 0, None, 0, 0):
        a, b, _, _, _, info = lapack.dtgexc(A0.copy(), B0.copy(), np.eye(m), np.eye(m), n1 + 1, 1)
        print(json.dumps({"window": T, "list_index": q, "row": j1 + j, "n1": n1, "n2": n2, "lapack_info": int(info),
                          "S_block": A0.tolist(), "T_block": B0.tolist()}))
        break
else:
    print("no rejection in the oracle replay of window", T)
print("2x2|2x2 swaps of the window that LAPACK dtgexc rejects on the same blocks:", lapack_rejects)
