"""Window-kernel phase profile (SN_WPROF=1): one config-2 reordering, phases per window."""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1905_04975_b200 as sn
from workloads import make_config
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = make_config(cfg, seed=1, device="cuda")
for it in range(2):
    S, Q = p.S.clone(), p.Q.clone()
    r = sn.reorder(S, Q, p.select, window=p.w, lookahead=0, q_stream_overlap=0)
    torch.cuda.synchronize()
    print("rc", r["rc"], "windows", r["stats"]["windows"], "ms", r["stats"]["ms_device"], flush=True)
