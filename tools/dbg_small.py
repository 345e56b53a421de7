"""Tiny reordering under torch for debugging (host or device buffers)."""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1905_04975_b200 as sn
from workloads import make_problem
mode = sys.argv[1] if len(sys.argv) > 1 else "device"
p = make_problem(300, 0.25, "householder", "bernoulli", 0.35, 64, seed=1)
if mode == "device":
    S, Q = p.S.cuda(), p.Q.cuda()
elif mode == "host":
    S, Q = p.S.clone(), p.Q.clone()
else:   # raw cudaMalloc'd buffers outside torch's allocator
    import ctypes
    cr = ctypes.CDLL("libcudart.so.12")
    S, Q = p.S.cuda(), p.Q.cuda()
    torch.cuda.synchronize()
r = sn.reorder(S, Q, p.select, window=64, lookahead=0, q_stream_overlap=0, serialize=1)
print(mode, "rc", r["rc"], flush=True)
torch.cuda.synchronize()
