"""Row f1 measurement: fused chain Q updates (opts.fuse_chain) against the default executor.

  python tools/fuse_chain_ab.py [--config 3] [--reps 3]

Alternates unfused / fused reorderings of the same BASELINE config (inputs copied from a
pristine device copy before each run, outside the timing), timing each on the device (the
library's CUDA events, sn_stats.ms_device); one more pair with opts.profile = 1 gives the
isolated Q-kernel time per run.  Checks the two results are bitwise equal.  One JSON line."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1905_04975_b200 as sn  # noqa: E402
from workloads import make_config  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    sn.build()
    p = make_config(args.config, seed=args.seed, device="cuda")
    S0, Q0 = p.S.contiguous(), p.Q.contiguous()
    S, Q = torch.empty_like(S0), torch.empty_like(Q0)
    times = {0: [], 1: []}
    qk = {}
    pairs = 0
    res = {}
    for rep in range(args.reps + 2):
        for fuse in (0, 1):
            S.copy_(S0); Q.copy_(Q0)
            torch.cuda.synchronize()
            prof = 1 if rep == args.reps + 1 else 0
            r = sn.reorder(S, Q, p.select, window=p.w, fuse_chain=fuse, profile=prof)
            torch.cuda.synchronize()
            assert r["rc"] == 0, r
            st = r["stats"]
            if prof:
                qk[fuse] = st["ms_kernel"][3]
            elif rep >= 1:
                times[fuse].append(st["ms_device"])
            if fuse:
                pairs = st["fused_q_pairs"]
            if rep == 0:
                res[fuse] = (S.clone(), Q.clone())
    bitwise = bool(torch.equal(res[0][0], res[1][0]) and torch.equal(res[0][1], res[1][1]))
    out = {"row": "f1_fused_chain_q", "config": args.config, "n": p.n, "w": p.w,
           "windows": r["stats"]["windows"], "levels": r["stats"]["levels"], "fused_q_pairs": pairs,
           "ms_unfused": times[0], "ms_fused": times[1],
           "median_unfused_ms": statistics.median(times[0]), "median_fused_ms": statistics.median(times[1]),
           "q_kernel_ms_isolated": {"unfused": qk.get(0), "fused": qk.get(1)},
           "bitwise_equal": bitwise}
    print(json.dumps(out))
    return 0 if bitwise else 1


if __name__ == "__main__":
    sys.exit(main())
