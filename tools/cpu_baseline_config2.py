"""The "CPU baseline, N cores" row of SURVEY §8d-5: the oracle's accumulated mode (the same
plain C, its independent panel rows / columns on all host threads via -fopenmp) over the whole
of BASELINE config 2 (n = 16 384, w = 256) on the GPU box's host cores.  One JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from workloads import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
threads = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
p = make_config(cfg, seed=1, device="cuda")
S = np.asfortranarray(p.S.cpu().numpy().T)
Q = np.asfortranarray(p.Q.cpu().numpy().T)
t0 = time.perf_counter()
r = oracle.reorder_threads(S, Q, p.select, p.w, threads, inplace=True)
dt = time.perf_counter() - t0
cpu = open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": \t") if os.path.exists("/proc/cpuinfo") else "?"
print(json.dumps({"row": "cpu_baseline_n_cores", "config": cfg, "n": p.n, "w": p.w, "rc": r["rc"],
                  "threads": threads, "cpu": cpu, "seconds": dt, "windows": r["stats"]["windows"],
                  "eq_flops": r["stats"]["eq_flops"], "gflops": r["stats"]["eq_flops"] / dt / 1e9,
                  "kind": "oracle mode (ii), -fopenmp build, full run"}), flush=True)
