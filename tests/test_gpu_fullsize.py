"""Full-size checks at BASELINE.json configs 3 (n = 40 000, the bench workload, in bench.py's
launch configuration) and 4 (n = 65 536, worst-case chain) on the GPU (-m gpu).

The oracle cannot run these sizes end to end, so the checks are the
properties that hold at any size (north_star invariants):
  * block map and selection mask bit-exact against the stable partition of the input blocks;
  * S exactly quasi-triangular (zero below the subdiagonal, subdiagonal only inside 2x2 blocks);
  * 1x1 eigenvalues bitwise equal along the permutation, 2x2 eigenvalues within 1e-10 relative;
  * sketched residual ||(A - Q S Q^T) X|| / ||A X|| and orthogonality ||(Q^T Q - I) X|| / ||X||
    with a Gaussian X of 16 columns (harness arithmetic: torch FP64 matmul), <= 100 n eps;
plus, for config 3, prefix parity with the oracle (the first 32 windows on both sides, >= 3 DAG
levels, all of S and Q compared elementwise within 1e-9 ||S||_F).
"""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1905_04975_b200 as sn
from tests.helpers import EPS, blocks_of, stable_partition
from workloads import make_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    sn.build()
    assert torch.cuda.is_available()


def _bmap_gpu(T):
    """Block map from the subdiagonal of S (T holds S^T: S[i+1, i] = T[i, i+1])."""
    sub = (T.diagonal(1) != 0).cpu().numpy()
    n = T.shape[0]
    bm = np.zeros(n, np.int8)
    i = 0
    while i < n - 1:
        if sub[i]:
            bm[i], bm[i + 1] = 1, 2
            i += 2
        else:
            i += 1
    return bm


def _block_eigs(a, b, c, d):
    """Eigenvalues of [[a, b], [c, d]] (vectorised), sorted by imaginary part."""
    tr = 0.5 * (a + d)
    disc = np.sqrt((0.5 * (a - d)) ** 2 + b * c + 0j)
    l1, l2 = tr + disc, tr - disc
    swap = l1.imag > l2.imag
    return np.where(swap, l2, l1), np.where(swap, l1, l2)


def _entries(T, rows, cols):
    """S[rows, cols] from the transposed storage."""
    return T[torch.as_tensor(cols, device=T.device), torch.as_tensor(rows, device=T.device)].cpu().numpy()


def _run_fullsize(cfg, prefix_windows=0, min_levels=1):
    p = make_config(cfg, seed=1, device="cuda")
    n = p.n
    S, Q = p.S, p.Q                      # row-major tensors holding S^T, Q^T
    bm0 = _bmap_gpu(S)
    b0 = blocks_of(bm0)
    rows0 = np.array([r for r, _ in b0])
    sizes = np.array([z for _, z in b0])
    flags = np.array([bool(p.select[r] or (z == 2 and p.select[r + 1])) for r, z in b0])
    diag0 = S.diagonal().cpu().numpy()
    r2 = rows0[sizes == 2]
    blk0 = [_entries(S, r2 + dr, r2 + dc) for dr, dc in ((0, 0), (0, 1), (1, 0), (1, 1))]
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.randn((n, 16), dtype=torch.float64, device="cuda", generator=g)
    AX = Q.t() @ (S.t() @ (Q @ X))       # A X = Q0 S0 Q0^T X
    nAX = torch.linalg.norm(AX).item()

    prefix = None
    if prefix_windows:
        S0h = np.asfortranarray(S.cpu().numpy().T)
        Q0h = np.asfortranarray(Q.cpu().numpy().T)
        Sp, Qp = S.clone(), Q.clone()
        got = sn.reorder(Sp, Qp, p.select, window=p.w, max_windows=prefix_windows)
        torch.cuda.synchronize()
        # the prefix must exercise the multi-level executor (lookahead strips, Q overlap)
        assert got["stats"]["levels"] >= min_levels, got["stats"]["levels"]
        # the oracle's panel rows / columns on the host's cores (bitwise the one-thread result,
        # tests/test_oracle_pins.py): the same arithmetic, minutes less of the GPU suite
        ref = oracle.reorder_threads(S0h, Q0h, p.select, w=p.w, threads=os.cpu_count() or 1,
                                     max_windows=prefix_windows, inplace=True)
        assert got["rc"] == 0 == ref["rc"]
        np.testing.assert_array_equal(got["bmap"], ref["bmap"])
        nS = float(torch.linalg.norm(S).item())
        dS = np.abs(Sp.cpu().numpy().T - ref["S"]).max()
        dQ = np.abs(Qp.cpu().numpy().T - ref["Q"]).max()
        prefix = (dS / nS, dQ)
        del Sp, Qp, S0h, Q0h, ref
        assert dS <= 1e-9 * nS and dQ <= 1e-9 * nS, prefix

    # the bench's launch configuration: default options, device buffers, its stream
    r = sn.reorder(S, Q, p.select, window=p.w)
    torch.cuda.synchronize()
    assert r["rc"] == 0
    # block map / selection: the stable partition, bit-exact
    order = stable_partition(sizes, flags)
    exp_bmap = np.concatenate([[0] if sizes[t] == 1 else [1, 2] for t in order]).astype(np.int8)
    np.testing.assert_array_equal(r["bmap"], exp_bmap)
    np.testing.assert_array_equal(_bmap_gpu(S), exp_bmap)
    m = int(sizes[flags].sum())
    assert r["m"] == m
    exp_sel = np.zeros(n, np.int32)
    exp_sel[:m] = 1
    np.testing.assert_array_equal(r["select"], exp_sel)
    # exactly quasi-triangular: S[i, j] = T[j, i] = 0 for i >= j + 2
    assert not bool((torch.triu(S, 2) != 0).any().item())
    # eigenvalues along the permutation
    b1 = blocks_of(exp_bmap)
    rows1 = np.array([rr for rr, _ in b1])
    diag1 = S.diagonal().cpu().numpy()
    one = sizes[order] == 1
    assert np.array_equal(diag1[rows1[one]], diag0[rows0[order][one]])   # bitwise
    two_new = rows1[~one]
    blk1 = [_entries(S, two_new + dr, two_new + dc) for dr, dc in ((0, 0), (0, 1), (1, 0), (1, 1))]
    # map each moved 2x2 block back to its input block
    inv = {int(rows0[t]): k for k, t in enumerate(np.where(sizes == 2)[0])}
    src = np.array([inv[int(rows0[t])] for t in order[~one]])
    e0a, e0b = _block_eigs(*[x[src] for x in blk0])
    e1a, e1b = _block_eigs(*blk1)
    scale = np.maximum(1.0, np.abs(e0a))
    assert np.max(np.maximum(np.abs(e1a - e0a), np.abs(e1b - e0b)) / scale) <= 1e-10
    # sketched invariants (c4 #15)
    res = torch.linalg.norm(Q.t() @ (S.t() @ (Q @ X)) - AX).item() / nAX
    orth = torch.linalg.norm(Q @ (Q.t() @ X) - X).item() / torch.linalg.norm(X).item()
    print("config%d: windows=%d levels=%d residual=%.3g orthogonality=%.3g prefix=%s"
          % (cfg, r["stats"]["windows"], r["stats"]["levels"], res, orth, prefix))
    assert res <= 100 * n * EPS and orth <= 100 * n * EPS
    return r


def test_config3_fullsize_bench_launch():
    # 32 windows of the schedule spanning several DAG levels, in the bench launch
    # configuration (lookahead and Q-stream overlap on), compared over all of S and Q
    _run_fullsize(3, prefix_windows=32, min_levels=3)


def test_config4_fullsize_worst_case_chain():
    _run_fullsize(4)


def test_config4_prefix_parity_sampled_Q():
    """Config 4 (n = 65 536, worst-case chain): the first 16 windows against the oracle, all of
    S and a 4 096-row sample of Q (or_reorder_q: Q's rows are updated independently; the full
    Q does not fit twice in host memory beside S), elementwise within 1e-9 ||S||_F."""
    p = make_config(4, seed=1, device="cuda")
    n, K = p.n, 16
    S, Q = p.S, p.Q
    rows = np.sort(np.random.default_rng(3).choice(n, 4096, replace=False))
    S0h = np.asfortranarray(S.cpu().numpy().T)                       # no copy: S^T row-major
    Q0s = np.asfortranarray(Q[:, torch.as_tensor(rows, device="cuda")].cpu().numpy().T)
    nS = float(torch.linalg.norm(S).item())
    got = sn.reorder(S, Q, p.select, window=p.w, max_windows=K)
    torch.cuda.synchronize()
    assert got["rc"] == 0 and got["stats"]["windows"] == K
    ref = oracle.reorder_threads(S0h, Q0s, p.select, w=p.w, threads=os.cpu_count() or 1, max_windows=K,
                                 inplace=True)
    assert ref["rc"] == 0 and ref["stats"]["windows"] == K
    np.testing.assert_array_equal(got["bmap"], ref["bmap"])
    dS = 0.0
    for c0 in range(0, n, 4096):                                       # column blocks of S
        blk = S[c0:c0 + 4096].cpu().numpy()                            # = S[:, c0:c0+4096]^T
        dS = max(dS, float(np.abs(blk - ref["S"][:, c0:c0 + 4096].T).max()))
    dQ = float(np.abs(Q[:, torch.as_tensor(rows, device="cuda")].cpu().numpy().T - ref["Q"]).max())
    print("config4 prefix K=%d levels=%d: max|dS|/||S||=%.3g max|dQ| (4096 rows)=%.3g"
          % (K, got["stats"]["levels"], dS / nS, dQ))
    assert dS <= 1e-9 * nS and dQ <= 1e-9 * nS
