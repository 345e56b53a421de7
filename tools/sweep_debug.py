import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_04975_b200 as sn
from workloads import make_hessenberg
n, ns, w, m = 1500, 40, 128, 12
h = make_hessenberg(n, ns, q="none", seed=6, device="cuda")
H1 = h.H.clone(); H2 = h.H.clone()
sn.qr_sweep(H1, None, h.sr, h.si, window=w, bulges_per_chain=m, lookahead=0)
sn.qr_sweep(H2, None, h.sr, h.si, window=w, bulges_per_chain=m, lookahead=1)
torch.cuda.synchronize()
A = H1.cpu().numpy().T; B = H2.cpu().numpy().T
D = np.abs(A - B) > 1e-10 * np.abs(A).max()
rows, cols = np.nonzero(D)
print("ndiff", D.sum())
if D.sum():
    print("rows", rows.min(), rows.max(), "cols", cols.min(), cols.max())
    # first differing entries
    idx = np.argsort(cols * n + rows)[:20]
    print(list(zip(rows[idx], cols[idx])))
os.environ["SN_SWEEP_ALLCRIT"] = "1"
H3 = h.H.clone()
sn.qr_sweep(H3, None, h.sr, h.si, window=w, bulges_per_chain=m, lookahead=1)
torch.cuda.synchronize()
print("allcrit ndiff", (np.abs(H3.cpu().numpy().T - A) > 1e-10 * np.abs(A).max()).sum())
del os.environ["SN_SWEEP_ALLCRIT"]
os.environ["SN_SWEEP_DBG_WAITW"] = "1"
H4 = h.H.clone()
sn.qr_sweep(H4, None, h.sr, h.si, window=w, bulges_per_chain=m, lookahead=1)
torch.cuda.synchronize()
print("waitW ndiff", (np.abs(H4.cpu().numpy().T - A) > 1e-10 * np.abs(A).max()).sum())
del os.environ["SN_SWEEP_DBG_WAITW"]
sc = sn.sweep_schedule(n, ns, w, m)

