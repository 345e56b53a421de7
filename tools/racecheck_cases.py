"""Smallest cases of every GPU path, for compute-sanitizer racecheck / synccheck / memcheck
(VERDICT r1 item 10): the reordering (window kernel, TMA panel kernels, cp.async fallback via
an odd leading dimension), the pencil path, the sweep, the eigenvectors."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1905_04975_b200 as sn  # noqa: E402
from workloads import make_hessenberg, make_pencil, make_problem  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "reorder"):
    p = make_problem(300, p2=0.25, q="householder", psel=0.4, w=64, seed=3)
    S, Q = p.S.cuda(), p.Q.cuda()
    print("reorder", sn.reorder(S, Q, p.select, window=64)["rc"], flush=True)
    S, Q = p.S.cuda(), p.Q.cuda()
    print("reorder w=256", sn.reorder(S, Q, p.select, window=256)["rc"], flush=True)
    n, ld = 200, 201
    p = make_problem(n, p2=0.25, q="householder", psel=0.4, w=64, seed=4)
    Sb = torch.zeros((n, ld), dtype=torch.float64); Qb = torch.zeros((n, ld), dtype=torch.float64)
    Sb[:, :n] = p.S; Qb[:, :n] = p.Q
    Sb, Qb = Sb.cuda(), Qb.cuda()
    sel = p.select.astype(np.int32).copy()
    print("reorder odd ld", sn.sn_reorder_schur(n, Sb.data_ptr(), ld, Qb.data_ptr(), ld, sel)[0], flush=True)
if which in ("all", "pencil"):
    g = make_pencil(200, p2=0.25, q="householder", psel=0.4, w=64, seed=5)
    dev = [x.cuda() for x in (g.S, g.T, g.Q, g.Z)]
    print("pencil", sn.reorder_pencil(*dev, g.select, window=64)["rc"], flush=True)
if which in ("all", "sweep"):
    h = make_hessenberg(300, 16, q="householder", seed=6, device="cuda")
    print("sweep staged", sn.qr_sweep(h.H.clone(), h.Q.clone(), h.sr, h.si, window=64, bulges_per_chain=8)["rc"], flush=True)
    print("sweep L2", sn.qr_sweep(h.H.clone(), h.Q.clone(), h.sr, h.si, window=256, bulges_per_chain=8)["rc"], flush=True)
if which in ("all", "eigvec"):
    p = make_problem(400, p2=0.25, q="householder", psel=0.5, w=64, seed=7)
    print("eigvec", sn.eigenvectors(p.S.cuda(), p.Q.cuda(), p.select)["rc"], flush=True)
torch.cuda.synchronize()
print("done")
