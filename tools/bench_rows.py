#!/usr/bin/env python
"""Measurement of the SURVEY §8 f-rows on one GPU (bench.py keeps the headline metric).

  python tools/bench_rows.py --row f2|f3|f4 [--steps K] [--warmup W] [--n N]

* f2 -- generalized reordering of a config-2-shaped pencil (n = 16 384, w = 256, 25 % 2x2
  blocks, Bernoulli(0.35), Q and Z random orthogonal): equivalent update flops per window
  2k^2 (2(n-j2) + 2j1 + n_Q + n_Z) per second (sn_reorder_pencil_ex).
* f3 -- one multishift QR sweep on a random n = 40 000 Hessenberg matrix with 256 shifts
  (LAPACK xLAQR0's shift count for n >= 6000) and a random orthogonal Q: equivalent update
  flops per window 2k^2 ((n-j2) + j1 + n) per second (sn_qr_sweep).
* f4 -- right eigenvectors of the selected eigenvalues of BASELINE config 3 (n = 40 000,
  Bernoulli(0.35) blocks, ~14 000 columns), back-transformed by the random orthogonal Q:
  algorithmic flops (back-substitution solves + update GEMMs + back-transform GEMM) per
  second (sn_eigenvectors).
Every step starts from a pristine device copy (restored outside the timed region); times are
CUDA events on the calling stream.  One JSON line per run.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1905_04975_b200 as sn  # noqa: E402
from workloads import make_config, make_hessenberg, make_pencil  # noqa: E402

FP64_PEAK_GFLOPS = 37074.0


def timed(fn, restore, steps, warmup):
    stream = torch.cuda.current_stream()
    out, times = None, []
    for it in range(warmup + steps):
        restore()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = fn(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        if it >= warmup:
            times.append(e0.elapsed_time(e1))
    return out, times


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--row", choices=["f2", "f3", "f4"], required=True)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--shifts", type=int, default=256)
    ap.add_argument("--window", type=int, default=0, help="f3: sweep window (0: library default)")
    ap.add_argument("--chain", type=int, default=0, help="f3: bulges per chain (0: library default)")
    args = ap.parse_args()
    sn.build()
    dev = torch.device("cuda", 0)
    line = {"row": args.row, "steps": args.steps, "warmup": args.warmup, "dtype": "f64", "data": "synthetic"}
    if args.row == "f2":
        n = args.n or 16384
        p = make_pencil(n, p2=0.25, q="householder", psel=0.35, w=256, seed=1, device=dev)
        src = [p.S, p.T, p.Q, p.Z]
        work = [x.clone() for x in src]

        def restore():
            for a, b in zip(work, src):
                a.copy_(b)
        r, times = timed(lambda s: sn.reorder_pencil(*work, p.select, window=256, stream=s.cuda_stream),
                         restore, args.steps, args.warmup)
        st = r["stats"]
        eq = st["eq_flops"]
        line.update(workload="pencil n=%d w=256 25%% 2x2 Bernoulli(0.35), Q and Z householder, seed 1" % n,
                    rc=r["rc"], windows=st["windows"], levels=st["levels"], swaps=st["swaps"])
    elif args.row == "f3":
        n = args.n or 40000
        h = make_hessenberg(n, args.shifts, q="householder", seed=1, device=dev)
        H, Q = h.H.clone(), h.Q.clone()

        def restore():
            H.copy_(h.H)
            Q.copy_(h.Q)
        kw = {}
        if args.window:
            kw["window"] = args.window
        if args.chain:
            kw["bulges_per_chain"] = args.chain
        r, times = timed(lambda s: sn.qr_sweep(H, Q, h.sr, h.si, stream=s.cuda_stream, **kw), restore, args.steps,
                         args.warmup)
        st = r["stats"]
        eq = st["eq_flops"]
        line.update(workload="random Hessenberg n=%d, %d random shifts (conjugate pairs), Q householder, seed 1"
                    % (n, len(h.sr)), rc=r["rc"], windows=st["windows"], levels=st["levels"],
                    chains=st["chains"], bulges=st["bulges"], opts=kw)
    else:
        p = make_config(3, seed=1, device=dev)
        sel = p.select.astype(np.int32)
        r, times = timed(lambda s: sn.eigenvectors(p.S, p.Q, sel, stream=s.cuda_stream), lambda: None,
                         args.steps, args.warmup)
        st = r["stats"]
        eq = st["flops_solve"] + st["flops_update"] + st["flops_backtransform"]
        line.update(workload="eigenvectors of the selected blocks of config 3 (n=40000, Bernoulli(0.35)), "
                             "back-transformed by Q", rc=r["rc"], columns=st["columns"], tiles=st["tiles"],
                    rescales=st["rescales"], ms_backsubstitution=st["ms_backsubstitution"],
                    ms_backtransform=st["ms_backtransform"], flops_update=st["flops_update"],
                    flops_backtransform=st["flops_backtransform"], flops_solve=st["flops_solve"])
    ms = float(np.mean(times))
    line.update(ms_per_step=ms, times_ms=times, flops=eq, value=eq / (ms / 1000.0) / 1e9, unit="GFLOP/s",
                frac_fp64_peak=eq / (ms / 1000.0) / 1e9 / FP64_PEAK_GFLOPS, launches=st.get("launches"))
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
