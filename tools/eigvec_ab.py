"""A/B of row f4 (sn_eigenvectors) between library builds (tools/build_variant.py copies).

  python tools/eigvec_ab.py [--reps 3] LIB [LIB ...]     (LIB = path or "default")

Each library in its own process (SN_LIB_PATH): the eigenvectors of config 3's selected blocks,
back-transformed by Q, timed on the device (events), the library's phase split, and a digest of
X and the scale exponents so the builds can be checked for bitwise equality.  One JSON line each."""
import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(reps):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_1905_04975_b200 as sn
    from workloads import make_config
    p = make_config(3, seed=1, device="cuda")
    sel = p.select.astype(np.int32)
    ms, st, dig = [], None, None
    for it in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s = torch.cuda.current_stream()
        e0.record(s)
        r = sn.eigenvectors(p.S, p.Q, sel, stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        assert r["rc"] == 0, r["rc"]
        if it >= 1:
            ms.append(e0.elapsed_time(e1))
        if it == 0:
            h = hashlib.sha1()
            h.update(r["X"].cpu().numpy().tobytes())
            h.update(np.asarray(r["scale_exp"]).tobytes() if r.get("scale_exp") is not None else b"")
            dig = h.hexdigest()[:16]
        st = r["stats"]
    print(json.dumps({"lib": os.path.basename(os.environ.get("SN_LIB_PATH", "default")), "row": "f4",
                      "ms": ms, "median_ms": statistics.median(ms),
                      "ms_backsubstitution": st["ms_backsubstitution"], "ms_backtransform": st["ms_backtransform"],
                      "rescales": st["rescales"], "launches": st.get("launches"), "digest": dig}), flush=True)


def main():
    if os.environ.get("SN_AB_CHILD"):
        child(int(os.environ["SN_AB_REPS"]))
        return 0
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    for lib in a.libs:
        env = dict(os.environ, SN_AB_CHILD="1", SN_AB_REPS=str(a.reps))
        if lib != "default":
            env["SN_LIB_PATH"] = os.path.abspath(lib)
        subprocess.run([sys.executable, os.path.abspath(__file__)], env=env, check=False)
    return 0


if __name__ == "__main__":
    sys.exit(main())
