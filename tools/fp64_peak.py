"""Measure the FP64 roofline denominators on the GPU box (harness tool).

cuBLAS DGEMM (torch.matmul fp64) 8192^3: best of 10 (burst) and back to back
for ~4 s (sustained), with nvidia-smi clocks sampled during the sustained loop.
Also times the panel shapes of the hot path (K = 256) for a cuBLAS bar.
Prints JSON lines.
"""
import json
import subprocess
import time

import torch


def clocks_start(path):
    return subprocess.Popen(
        ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
         "--format=csv,noheader,nounits", "-lms", "200"],
        stdout=open(path, "w"), stderr=subprocess.DEVNULL)


def main():
    dev = torch.device("cuda:0")
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = torch.empty_like(a)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"probe": "cublas_dgemm_burst", "n": n, "ms": best, "tflops": 2 * n**3 / best / 1e9}))
    p = clocks_start("gpurun_out/clocks_dgemm.csv")
    time.sleep(0.5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 0
    t0 = time.time()
    while time.time() - t0 < 4.0:
        for _ in range(4):
            torch.matmul(a, b, out=c)
        reps += 4
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    p.terminate()
    print(json.dumps({"probe": "cublas_dgemm_sustained", "n": n, "reps": reps, "tflops": 2 * n**3 * reps / ms / 1e9}))
    try:
        rows = [r.split(",") for r in open("gpurun_out/clocks_dgemm.csv").read().strip().splitlines()]
        sm = sorted(float(r[0]) for r in rows if r and r[0].strip().replace('.', '').isdigit())
        print(json.dumps({"probe": "clocks_dgemm", "sm_mhz_median": sm[len(sm) // 2] if sm else None,
                          "samples": len(sm)}))
    except Exception as exc:  # noqa: BLE001
        print(json.dumps({"probe": "clocks_dgemm", "error": str(exc)}))
    # panel shapes: Z^T (256x256) @ P (256 x 40000), and P (40000x256) @ Z
    k, N = 256, 40000
    z = torch.randn(k, k, dtype=torch.float64, device=dev)
    pl = torch.randn(k, N, dtype=torch.float64, device=dev)
    pr = torch.randn(N, k, dtype=torch.float64, device=dev)
    for name, fn in (("left_ZtP", lambda: torch.matmul(z.t(), pl)), ("right_PZ", lambda: torch.matmul(pr, z))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(json.dumps({"probe": "cublas_panel_" + name, "k": k, "N": N, "ms": ms,
                          "tflops": 2 * k * k * N / ms / 1e9}))


if __name__ == "__main__":
    main()
