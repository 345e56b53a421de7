#!/usr/bin/env python
"""Benchmark of the B200 Schur-reordering hot path (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl sn|reference]

A step is one full reordering (all rows of SURVEY §8a: structure scan, schedule, window
tasks, left/right/Q updates) of BASELINE config C (default 3: n = 40000, w = 256, 25% 2x2
blocks, Bernoulli(0.35) selection, random orthogonal Q) with S and Q resident in HBM.  Each
step starts from the same pristine input (restored by a device copy outside the timed
region).  Inputs (2 x 12.8 GB) exceed L2 (126 MB), so no extra flush is needed.

metric: FP64 GFLOP/s of the equivalent update flops and wall seconds.
Rank 0 prints one JSON line.  For N > 1 (torchrun, one process per GPU) the SAME problem is
sharded over the ranks (sn_reorder_schur_dist: S column blocks of width
--col-block, Q row blocks, each window's Z broadcast by NCCL): scaling "strong", time = max
over ranks of the device time.  --emulate-ranks P runs the sharded program for P ranks on
one GPU (sn_reorder_schur_dist_local; a measurement of the sharded path's overheads, not a
multi-GPU number).  --impl reference times the CPU oracle (oracle/, plain C, 1 core) on a
bounded prefix of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Schur reordering GFLOP/s FP64 & wall s at n=40000"
FP64_PEAK_GFLOPS = 37074.0   # measured DMMA m16n8k8.f64 peak, profiles/r01_fp64_peaks.jsonl


def dist_setup(ngpus):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        torch.cuda.set_device(local)
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(ws, x):
    if ws == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class Clocks:
    """nvidia-smi sampler for the timed region (SM clock, max, throttle reasons)."""

    def __init__(self, idx):
        self.path = os.path.join(ROOT, "gpurun_out", "bench_clocks_%d.csv" % idx)
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        self.p = None
        self.idx = idx

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()

    def summary(self):
        try:
            rows = [r.split(", ") for r in open(self.path).read().strip().splitlines()]
            rows = [r for r in rows if len(r) >= 7]
            sm = sorted(float(r[0]) for r in rows)
            reasons = set()
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for r in rows:
                for nm, v in zip(names, r[3:7]):
                    if v.strip() == "Active":
                        reasons.add(nm)
            return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                    "sm_max_mhz": float(rows[0][1]) if rows else None,
                    "reasons": sorted(reasons), "samples": len(rows)}
        except Exception as exc:  # noqa: BLE001
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": str(exc)}


def workload_desc(cfg, prob):
    m = prob.meta
    return ("config%d: n=%d, w=%d, %d blocks (%d 2x2), selection %s%s, Q %s, seed %d"
            % (cfg, m["n"], m["w"], m["blocks"], m["blocks_2x2"], m["sel"],
               "" if m["psel"] is None else "(%.2f)" % m["psel"], m["q"], m["seed"]))


def oracle_sample(prob, target_gflop, device_S0, device_Q0):
    """Time the CPU oracle (mode ii, 1 core) on the first K windows of the workload."""
    import oracle   # the reference arm touches only oracle/ (sample sizing included)
    S = np.asfortranarray(device_S0.cpu().numpy().T)
    Q = np.asfortranarray(device_Q0.cpu().numpy().T)
    sub = np.diag(S, -1) != 0.0
    bm = np.zeros(prob.n, np.int8)
    i = 0
    while i < prob.n - 1:
        if sub[i]:
            bm[i], bm[i + 1] = 1, 2
            i += 2
        else:
            i += 1
    sel8 = np.zeros(prob.n, np.int8)
    i = 0
    while i < prob.n:
        s = 2 if bm[i] == 1 else 1
        sel8[i:i + s] = 1 if prob.select[i:i + s].any() else 0
        i += s
    sch = oracle.schedule(bm, sel8, prob.w)
    k, j1 = (sch["j2"] - sch["j1"]).astype(float), sch["j1"].astype(float)
    fl = 2 * k * k * ((prob.n - j1 - k) + j1 + prob.n)
    K = int(max(1, np.searchsorted(np.cumsum(fl), target_gflop * 1e9)))
    t0 = time.perf_counter()
    r = oracle.reorder(S, Q, prob.select, w=prob.w, mode=1, max_windows=K, inplace=True)
    dt = time.perf_counter() - t0
    assert r["rc"] == 0
    return {"gflops": r["stats"]["eq_flops"] / dt / 1e9, "seconds": dt, "windows": K,
            "eq_flops": r["stats"]["eq_flops"]}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on this box's host cores."""
    ws, rank, local = dist_setup(args.gpus)
    if rank != 0:
        return 0
    from workloads import make_config
    prob = make_config(args.config, seed=args.seed, device="cuda")
    vals = []
    info = None
    for it in range(args.warmup + args.steps):
        info = oracle_sample(prob, args.oracle_gflop, prob.S, prob.Q)
        if it >= args.warmup:
            vals.append(info)
    gf = sum(v["eq_flops"] for v in vals) / sum(v["seconds"] for v in vals) / 1e9
    sample = "first %d windows (schedule order) of %s; oracle mode (ii), naive triple loops" % (
        info["windows"], workload_desc(args.config, prob))
    line = {"impl": "reference", "metric": METRIC, "value": gf, "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * sum(v["seconds"] for v in vals) / len(vals),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_desc(args.config, prob), "sample": sample},
            "cpu_baseline": {"value": gf, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": gf, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_sharded(args, ws, rank, local):
    """N > 1: the sharded reordering of one problem over the ranks (strong scaling)."""
    import paper_1905_04975_b200 as sn
    from workloads import make_config
    dev = torch.device("cuda", local)
    prob = make_config(args.config, seed=args.seed, device=dev)
    n, bc = prob.n, args.col_block
    emu = ws == 1
    P = args.emulate_ranks if emu else ws
    ranks = list(range(P)) if emu else [rank]
    shards = [sn.shard(prob.S, prob.Q, P, bc, r) for r in ranks]
    S0 = [s for s, _ in shards]
    Q0 = [q for _, q in shards]
    del shards
    prob.S = prob.Q = None
    torch.cuda.empty_cache()
    S = [x.clone() for x in S0]
    Q = [x.clone() for x in Q0]
    if not emu:
        sn.dist_init(rank, ws, local)
    stream = torch.cuda.current_stream(dev)

    def call(Sl, Ql, **kw):
        if emu:
            return sn.reorder_dist_local(Sl, Ql, prob.select, n, bc, window=prob.w, stream=stream.cuda_stream, **kw)
        return sn.reorder_dist(Sl[0], Ql[0], prob.select, n, bc, window=prob.w, stream=stream.cuda_stream, **kw)

    def step():
        for a, b in zip(S, S0):
            a.copy_(b)
        for a, b in zip(Q, Q0):
            a.copy_(b)
        torch.cuda.synchronize(dev)
        barrier(ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = call(S, Q)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        assert r["rc"] == 0, r["rc"]
        return e0.elapsed_time(e1), r

    for _ in range(args.warmup):
        step()
    times, results = [], []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            ms, r = step()
            times.append(ms)
            results.append(r)
    clocks = clk.summary()
    tot_ms = allmax(ws, sum(times))
    st = results[-1]["stats"]
    eq = st["eq_flops"]
    value = eq * args.steps / (tot_ms / 1000.0) / 1e9
    gpu_launches = int(sum(sum(r["stats"]["launches"]) for r in results) / args.steps)
    e2e = None
    if args.e2e_steps > 0 and not emu:
        Sh = torch.empty(S0[0].shape, dtype=torch.float64, pin_memory=True)
        Qh = torch.empty(Q0[0].shape, dtype=torch.float64, pin_memory=True)
        et = []
        for _ in range(args.e2e_steps):
            Sh.copy_(S0[0]); Qh.copy_(Q0[0])
            torch.cuda.synchronize(dev)
            barrier(ws)
            t0 = time.perf_counter()
            r = sn.reorder_dist(Sh, Qh, prob.select, n, bc, window=prob.w)
            t1 = time.perf_counter()
            assert r["rc"] == 0
            et.append(t1 - t0)
        e2e_s = allmax(ws, sum(et))
        nb = 8 * (Sh.numel() + Qh.numel())
        e2e = {"value": eq * args.e2e_steps / e2e_s / 1e9, "unit": "GFLOP/s", "wall_s": e2e_s / args.e2e_steps,
               "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb, "note": "per rank bytes (its shards)"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "wall_s": tot_ms / args.steps / 1000.0,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_desc(args.config, prob),
                       "parallelism": ("emulated %d ranks on 1 GPU" % P) if emu else "sharded S col-blocks/Q row-blocks x%d" % ws,
                       "col_block": bc,
                       "l2": "inputs > 126 MB L2, no flush needed",
                       "windows": st["windows"], "levels": st["levels"], "swaps": st["swaps"],
                       "eq_tflop": eq / 1e12},
            "roofline": None,
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    if not emu:
        sn.dist_finalize()
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impl", default="sn", choices=["sn", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--oracle-gflop", type=float, default=40.0, help="size of the oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--col-block", type=int, default=1024, help="column block width of the sharded S")
    ap.add_argument("--emulate-ranks", type=int, default=0, help="sharded program for P ranks on one GPU")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    ws, rank, local = dist_setup(args.gpus)
    import paper_1905_04975_b200 as sn
    from workloads import make_config
    sn.lib()
    if ws > 1 or args.emulate_ranks > 0:
        return run_sharded(args, ws, rank, local)
    dev = torch.device("cuda", local)
    prob = make_config(args.config, seed=args.seed, device=dev)
    S0, Q0 = prob.S, prob.Q
    S, Q = torch.empty_like(S0), torch.empty_like(Q0)
    stream = torch.cuda.current_stream(dev)

    def step(profile, **kw):
        S.copy_(S0)
        Q.copy_(Q0)
        torch.cuda.synchronize(dev)
        barrier(ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = sn.reorder(S, Q, prob.select, window=prob.w, profile=profile, stream=stream.cuda_stream, **kw)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        assert r["rc"] == 0, r["rc"]
        return e0.elapsed_time(e1), r

    for _ in range(args.warmup):
        step(0)
    times, results = [], []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            ms, r = step(1)
            times.append(ms)
            results.append(r)
    clocks = clk.summary()
    tot_ms = allmax(ws, sum(times))
    st = results[-1]["stats"]
    eq = st["eq_flops"]
    value = ws * eq * args.steps / (tot_ms / 1000.0) / 1e9
    ms_per_step = tot_ms / args.steps
    # Per-kernel event times inside the timed region overlap (three streams), so each kind's
    # summed event time includes waiting for SMs held by the others (kernel_share below).  The
    # roofline of the dominant kind is taken from one extra step AFTER the timed region with
    # every launch on one stream (lookahead and Q overlap off): isolated launch durations.
    kinds = {0: "window", 1: "left_update", 2: "right_update", 3: "q_update", 4: "scan"}
    msk = [sum(r["stats"]["ms_kernel"][q] for r in results) for q in range(5)]
    share = {kinds[q]: msk[q] / sum(times) for q in range(5)}
    iso_ms, riso = step(1, lookahead=0, q_stream_overlap=0)
    msi = riso["stats"]["ms_kernel"]
    dom = max((1, 2, 3), key=lambda q: msi[q])
    # achieved = flops the kernel executes (the dense products minus the K steps where Z is
    # structurally zero) per second; the dense-equivalent rate is reported beside it
    ach = riso["stats"]["flops_exec_kernel"][dom] / (msi[dom] / 1000.0) / 1e12
    ach_eq = riso["stats"]["flops_kernel"][dom] / (msi[dom] / 1000.0) / 1e12
    ach_conc = sum(r["stats"]["flops_kernel"][dom] for r in results) / (msk[dom] / 1000.0) / 1e12
    launches_dom = riso["stats"]["launches"][dom]
    iso_share = {kinds[q]: msi[q] / iso_ms for q in range(5)}
    traffic, traffic_note = None, None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile)).get(kinds[dom])
        if tj:
            traffic = tj["dram_bytes_per_launch"]
            traffic_note = tj["note"]
    gpu_launches = int(sum(sum(r["stats"]["launches"]) for r in results) / args.steps)

    # e2e through the C ABI with host buffers (H2D + D2H inside the call).  The device work
    # copies are released first: the call stages S and Q in device memory of its own (at
    # config 4, 2 x 34 GB; with the pristine and work copies resident that would not fit)
    e2e = None
    if args.e2e_steps > 0:
        del S, Q
        torch.cuda.empty_cache()
        Sh = torch.empty(S0.shape, dtype=S0.dtype, pin_memory=True)
        Qh = torch.empty(Q0.shape, dtype=Q0.dtype, pin_memory=True)
        et = []
        for _ in range(args.e2e_steps):
            Sh.copy_(S0); Qh.copy_(Q0)
            torch.cuda.synchronize(dev)
            barrier(ws)
            t0 = time.perf_counter()
            r = sn.reorder(Sh, Qh, prob.select, window=prob.w)
            t1 = time.perf_counter()
            assert r["rc"] == 0
            et.append(t1 - t0)
        e2e_s = allmax(ws, sum(et))
        nbytes = 2 * 8 * prob.n * prob.n
        e2e = {"value": ws * eq * args.e2e_steps / e2e_s / 1e9, "unit": "GFLOP/s",
               "wall_s": e2e_s / args.e2e_steps, "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes}
        del Sh, Qh

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        info = oracle_sample(prob, args.oracle_gflop, S0, Q0)
        cpu = {"value": info["gflops"], "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
               "sample": "first %d windows (schedule order) of this workload, oracle mode (ii), %.1f s"
                         % (info["windows"], info["seconds"])}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "wall_s": ms_per_step / 1000.0,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_desc(args.config, prob), "parallelism": "replicas" if ws > 1 else "1gpu",
                       "l2": "inputs 2 x %.1f GB > 126 MB L2, no flush needed" % (8 * prob.n ** 2 / 1e9),
                       "windows": st["windows"], "levels": st["levels"], "swaps": st["swaps"],
                       "eq_tflop": eq / 1e12},
            "roofline": {"bound": "tensor", "kernel": kinds[dom], "achieved": ach * 1000.0,
                         "peak": FP64_PEAK_GFLOPS, "unit": "GFLOP/s", "frac": ach * 1000.0 / FP64_PEAK_GFLOPS,
                         "peak_source": "measured FP64 DMMA probe (MEASURED_PEAKS.json has no FP64 entry)",
                         "timing": "isolated launches: one extra serialized step after the timed region",
                         "achieved_dense_equivalent": ach_eq * 1000.0,
                         "executed_over_dense": riso["stats"]["flops_exec_kernel"][dom] / max(1.0, riso["stats"]["flops_kernel"][dom]),
                         "achieved_in_timed_region": ach_conc * 1000.0,
                         "launches": launches_dom, "traffic": traffic, "traffic_note": traffic_note},
            "kernel_share": share,
            "kernel_share_isolated": iso_share,
            "isolated_step_ms": iso_ms,
            "kernel_ms_isolated": {kinds[q]: msi[q] for q in range(5)},
            "clocks": clocks,
            "e2e": e2e,
            "gpu_launches": gpu_launches,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
