"""One config-3 reordering (bench launch options + per-launch events) with SN_TIMELINE set;
writes the launch timeline CSV and prints tools/timeline_summary.py's overlap summary."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1905_04975_b200 as sn  # noqa: E402
from workloads import make_config  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "timeline_config3.csv")
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = make_config(cfg, seed=1, device="cuda")
S, Q = p.S.clone(), p.Q.clone()
sn.reorder(S, Q, p.select, window=p.w)            # warm-up
S.copy_(p.S); Q.copy_(p.Q)
torch.cuda.synchronize()
os.environ["SN_TIMELINE"] = out
r = sn.reorder(S, Q, p.select, window=p.w, profile=1)
torch.cuda.synchronize()
print("rc", r["rc"], "ms_device", r["stats"]["ms_device"])
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "timeline_summary.py"), out])
