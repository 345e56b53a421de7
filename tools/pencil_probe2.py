"""Probe of a pencil rejection: the GPU's rejected swap (SN_DEBUG) and the oracle's verdict on
the same schedule prefix (run on the GPU box)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SN_DEBUG"] = "1"
import numpy as np, torch
import oracle, paper_1905_04975_b200 as sn
from workloads import make_pencil
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
p = make_pencil(n, p2=0.25, q="householder", psel=0.35, w=256, seed=1, device="cuda")
src = [p.S, p.T, p.Q, p.Z]
work = [x.clone() for x in src]
r = sn.reorder_pencil(*work, p.select, window=256)
torch.cuda.synchronize()
print("gpu rc", r["rc"], {k: r["stats"][k] for k in ("windows", "swaps", "rejected_window", "rejected_row", "rejected_n1", "rejected_n2")}, flush=True)
if r["rc"] == 1:
    K = r["stats"]["rejected_window"] + 1
    S, T = p.np("S"), p.np("T")
    t = time.time()
    ref = oracle.greorder(S, T, None, None, p.select, w=256, mode=1, max_windows=K)
    print("oracle rc", ref["rc"], ref["stats"], "%.1f s" % (time.time() - t), flush=True)
    j = r["stats"]["rejected_row"]
    # the oracle state before its rejection / after K windows around the GPU's rejected row
    np.savez("gpurun_out/pencil_probe_blocks.npz", S=ref["S"][j - 2:j + 6, j - 2:j + 6], T=ref["T"][j - 2:j + 6, j - 2:j + 6], j=j)
