"""A/B of window-kernel variants (prebuilt library copies, tools/build_variant.py).

  python tools/window_ab.py [--configs 2 3] [--reps 3] LIB [LIB ...]

Each library runs in its own process (SN_LIB_PATH): per config, `reps` default reorderings
timed on the device (sn_stats.ms_device, medians), one with opts.profile = 1 (isolated window
kernel time, kind 0), and a digest of the resulting S and Q so the variants can be checked for
bitwise equality.  One JSON line per (library, config)."""
import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(cfg, reps):
    sys.path.insert(0, ROOT)
    import torch
    import paper_1905_04975_b200 as sn
    from workloads import make_config
    p = make_config(cfg, seed=1, device="cuda")
    S0, Q0 = p.S.contiguous(), p.Q.contiguous()
    S, Q = torch.empty_like(S0), torch.empty_like(Q0)
    ms, digest, wk = [], None, None
    for rep in range(reps + 2):
        S.copy_(S0); Q.copy_(Q0)
        torch.cuda.synchronize()
        prof = 1 if rep == reps + 1 else 0
        r = sn.reorder(S, Q, p.select, window=p.w, profile=prof)
        torch.cuda.synchronize()
        assert r["rc"] == 0, r["rc"]
        if prof:
            wk = r["stats"]["ms_kernel"]
        elif rep >= 1:
            ms.append(r["stats"]["ms_device"])
        if rep == 0:
            h = hashlib.sha1()
            h.update(S.cpu().numpy().tobytes()); h.update(Q.cpu().numpy().tobytes())
            digest = h.hexdigest()[:16]
    print(json.dumps({"lib": os.path.basename(os.environ.get("SN_LIB_PATH", "default")), "config": cfg,
                      "ms_device": ms, "median_ms": statistics.median(ms),
                      "ms_kernel_isolated": wk, "window_ms_isolated": wk[0], "digest": digest}), flush=True)


def main():
    if os.environ.get("SN_AB_CHILD"):
        child(int(os.environ["SN_AB_CHILD"]), int(os.environ["SN_AB_REPS"]))
        return 0
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[2, 3])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    for cfg in a.configs:
        for lib in a.libs:
            env = dict(os.environ, SN_AB_CHILD=str(cfg), SN_AB_REPS=str(a.reps))
            if lib != "default":
                env["SN_LIB_PATH"] = os.path.abspath(lib)
            subprocess.run([sys.executable, os.path.abspath(__file__)], env=env, check=False)
    return 0


if __name__ == "__main__":
    sys.exit(main())
