"""Timing of the generalized (pencil) reordering, row f2 (a profile record, not the bench.py
contract): one seeded pencil of a BASELINE config's shape (make_pencil), W warm-up runs and K
timed runs from fresh copies, CUDA events on the call's stream.  Prints one JSON line.

  python tools/bench_pencil.py [--config 2] [--steps 2] [--warmup 1]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1905_04975_b200 as sn  # noqa: E402
from workloads import CONFIGS, make_pencil  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--cluster", type=int, default=0, help="opts.pencil_cluster (0 auto, 1 one CTA)")
    args = ap.parse_args()
    c = CONFIGS[args.config]
    p = make_pencil(c["n"], c["p2"], c["q"], c["sel"], c["psel"], c["w"], seed=1, device="cuda")
    sn.build()
    stream = torch.cuda.current_stream()
    times, st = [], None
    for it in range(args.warmup + args.steps):
        S, T, Q, Z = p.S.clone(), p.T.clone(), p.Q.clone(), p.Z.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = sn.reorder_pencil(S, T, Q, Z, p.select, window=c["w"], pencil_cluster=args.cluster)
        e1.record(stream)
        torch.cuda.synchronize()
        if r["rc"] != 0:
            st = r["stats"]
            print(json.dumps({"probe": "pencil_reorder", "rc": r["rc"], "rejected_window": st["rejected_window"],
                              "rejected_row": st["rejected_row"], "n1": st["rejected_n1"], "n2": st["rejected_n2"],
                              "windows": st["windows"], "swaps": st["swaps"]}))
            return
        if it >= args.warmup:
            times.append(e0.elapsed_time(e1))
            st = r["stats"]
    ms = sum(times) / len(times)
    print(json.dumps({
        "probe": "pencil_reorder", "config": "config%d pencil (make_pencil): n=%d, w=%d" % (args.config, c["n"], c["w"]),
        "ms": ms, "eq_tflop": st["eq_flops"] / 1e12, "tflops_equivalent": st["eq_flops"] / (ms * 1e9),
        "windows": st["windows"], "levels": st["levels"], "swaps": st["swaps"],
        "ms_device": st["ms_device"], "launches": st["launches"], "pencil_cluster": args.cluster,
        "times_ms": times}))


if __name__ == "__main__":
    main()
