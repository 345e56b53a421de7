"""A/B bitwise check of the pencil path between two builds of the library (tooling, GPU):
python tools/pencil_ab_bitwise.py OUT.npz [--cluster C]  (run once per build, SN_LIB_PATH
selecting the build), then python tools/pencil_ab_bitwise.py --compare A.npz B.npz."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402


def main():
    if sys.argv[1] == "--compare":
        a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
        bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
        print("bitwise equal" if not bad else "DIFFER: %s" % bad, {k: float(np.abs(a[k] - b[k]).max()) for k in a.files})
        return
    import torch
    import paper_1905_04975_b200 as sn
    from workloads import make_pencil
    cl = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    out = {}
    for n, w, p2, seed in ((700, 256, 0.25, 7), (2000, 128, 0.5, 12), (4096, 128, 0.25, 1)):
        p = make_pencil(n, p2=p2, q="householder", psel=0.35, w=w, seed=seed, device="cuda")
        S, T, Q, Z = p.S.clone(), p.T.clone(), p.Q.clone(), p.Z.clone()
        kw = {} if os.environ.get("SN_LIB_PATH", "").endswith("_base.so") else {"pencil_cluster": cl}
        r = sn.reorder_pencil(S, T, Q, Z, p.select, window=w, **kw)
        torch.cuda.synchronize()
        assert r["rc"] == 0, r["rc"]
        for k, X in (("S", S), ("T", T), ("Q", Q), ("Z", Z)):
            out["%s_%d" % (k, n)] = X.cpu().numpy()
    np.savez(sys.argv[1], **out)
    print("saved", sys.argv[1])


if __name__ == "__main__":
    main()
