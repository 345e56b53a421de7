"""Sharded-path statistics on one GPU (emulated ranks): schedule/plan time vs device time."""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1905_04975_b200 as sn
from workloads import make_config
cfg, P, bc = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
p = make_config(cfg, seed=1, device="cuda")
sh = [sn.shard(p.S, p.Q, P, bc, r) for r in range(P)]
S0 = [a for a, _ in sh]; Q0 = [b for _, b in sh]
for it in range(2):
    S = [x.clone() for x in S0]; Q = [x.clone() for x in Q0]
    torch.cuda.synchronize()
    r = sn.reorder_dist_local(S, Q, p.select, p.n, bc, window=p.w)
    st = r["stats"]
    print("dist P=%d bc=%d: ms_schedule %.1f ms_device %.1f ms_total %.1f launches %s" % (
        P, bc, st["ms_schedule"], st["ms_device"], st["ms_total"], st["launches"]), flush=True)
S, Q = p.S.clone(), p.Q.clone()
for it in range(2):
    S.copy_(p.S); Q.copy_(p.Q)
    r = sn.reorder(S, Q, p.select, window=p.w)
    st = r["stats"]
    print("single: ms_schedule %.1f ms_device %.1f ms_total %.1f" % (st["ms_schedule"], st["ms_device"], st["ms_total"]), flush=True)
