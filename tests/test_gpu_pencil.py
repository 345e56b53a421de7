"""GPU parity of the generalized reordering (-m gpu, through the C ABI).

The CUDA path (sn_reorder_pencil_ex: the window kernel with the pencil swap and the TMA panel
kernels on S, T, Q, Z) against the oracle's windowed generalized reordering (or_greorder mode
1, pinned to LAPACK dtgexc / dtgsen in tests/test_oracle_generalized.py) on the same seeded
pencils: block map and selection bit-exact, S, T, Q, Z elementwise within 1e-9 ||S||_F (the
in-window swap order differs, reading R12, so agreement is to rounding; the basis-sign
convention G7 makes the signs a function of the data, not of rounding-level choices such as
which re-triangularisation G2 keeps), and the invariants of a generalized reordering.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1905_04975_b200 as sn
from tests.helpers import blocks_of, bmap_from_S, stable_partition
from tests.test_oracle_generalized import check_greordering, check_gstructure
from workloads import make_pencil

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    sn.build()
    assert torch.cuda.is_available()


def _dev(X):
    return None if X is None else torch.as_tensor(np.ascontiguousarray(X.T)).cuda()


def _host(t):
    return None if t is None else t.cpu().numpy().T.copy(order="F")


def _run(p, window, with_q=True, with_z=True, **opts):
    S, T = p.np("S"), p.np("T")
    Q = p.np("Q") if with_q else None
    Z = p.np("Z") if with_z else None
    dS, dT, dQ, dZ = _dev(S), _dev(T), _dev(Q), _dev(Z)
    torch.cuda.synchronize()
    r = sn.reorder_pencil(dS, dT, dQ, dZ, p.select, window=window, **opts)
    torch.cuda.synchronize()
    r.update(S=_host(dS), T=_host(dT), Q=_host(dQ), Z=_host(dZ))
    return (S, T, Q, Z), r


def _compare(p, window, oracle_threads=0, **kw):
    (S, T, Q, Z), r = _run(p, window, **kw)
    ref = oracle.greorder(S, T, Q, Z, p.select, w=window, mode=1, threads=oracle_threads)
    assert r["rc"] == 0 == ref["rc"]
    assert r["m"] == ref["m"]
    np.testing.assert_array_equal(r["bmap"], ref["bmap"])
    np.testing.assert_array_equal(r["select"], ref["select"])
    nS, nT = np.linalg.norm(S), np.linalg.norm(T)
    worst = 0.0
    for key, nrm in (("S", nS), ("T", nT), ("Q", max(nS, 1.0)), ("Z", max(nS, 1.0))):
        if r[key] is not None:
            d = np.abs(r[key] - ref[key]).max() / nrm
            worst = max(worst, d)
            assert d <= 1e-9, (key, d)
    print("pencil n=%d: max elementwise diff / norm = %.3g" % (S.shape[0], worst))
    if Q is not None and Z is not None:
        check_greordering(S, T, Q, Z, p.select, r)
    else:
        check_gstructure(r["S"], r["T"])
    return r


@pytest.mark.parametrize("n,p2,w,psel,seed", [
    (40, 0.25, 16, 0.5, 1), (97, 0.0, 16, 0.35, 2), (150, 0.5, 32, 0.35, 3), (257, 0.25, 64, 0.35, 4),
    (300, 0.25, 256, 0.35, 5), (513, 0.5, 128, 0.5, 6), (700, 0.25, 256, 0.2, 7)])
def test_pencil_matches_oracle(n, p2, w, psel, seed):
    p = make_pencil(n, p2=p2, q="householder", psel=psel, w=w, seed=seed)
    r = _compare(p, w)
    assert r["stats"]["windows"] > 0 and r["stats"]["swaps"] > 0


def test_pencil_config1_size():
    # config-1 shape (n = 4096, w = 128, 25 % 2x2 blocks, Bernoulli(0.35)) as a pencil
    p = make_pencil(4096, p2=0.25, q="householder", psel=0.35, w=128, seed=1)
    r = _compare(p, 128, oracle_threads=os.cpu_count() or 1)   # bitwise the one-thread oracle
    print("pencil n=4096: windows=%d levels=%d swaps=%d ms_device=%.1f"
          % (r["stats"]["windows"], r["stats"]["levels"], r["stats"]["swaps"], r["stats"]["ms_device"]))


def test_pencil_without_q_or_z():
    p = make_pencil(200, p2=0.25, q="householder", psel=0.4, w=32, seed=8)
    _compare(p, 32, with_q=False)
    _compare(p, 32, with_z=False)
    _compare(p, 32, with_q=False, with_z=False)


@pytest.mark.parametrize("n", [0, 1, 2, 3])
def test_pencil_edge_sizes(n):
    p = make_pencil(max(n, 1), p2=0.5, q="householder", sel="all", w=16, seed=9)
    if n == 0:
        e = torch.zeros((0, 0), dtype=torch.float64, device="cuda")
        r = sn.reorder_pencil(e, e, e, e, np.zeros(0, np.int32), window=16)
        assert r["rc"] == 0 and r["m"] == 0
        return
    (S, T, Q, Z), r = _run(p, 16)
    assert r["rc"] == 0
    np.testing.assert_array_equal(r["S"], S)     # nothing to move: bitwise no-op
    np.testing.assert_array_equal(r["T"], T)


def test_pencil_trivial_selection_is_noop():
    p = make_pencil(300, p2=0.25, q="householder", sel="none", psel=None, w=64, seed=10)
    (S, T, Q, Z), r = _run(p, 64)
    assert r["rc"] == 0 and r["stats"]["windows"] == 0
    for a, b in ((S, r["S"]), (T, r["T"]), (Q, r["Q"]), (Z, r["Z"])):
        np.testing.assert_array_equal(a, b)


def test_pencil_forced_rejection_leaves_valid_form():
    p = make_pencil(400, p2=0.25, q="householder", psel=0.4, w=64, seed=11)
    (S, T, Q, Z), r = _run(p, 64, force_reject_window=3, force_reject_swap=40)
    assert r["rc"] == 1
    assert r["stats"]["rejected_window"] == 3
    bm = check_gstructure(r["S"], r["T"])
    np.testing.assert_array_equal(bm, r["bmap"])
    n = S.shape[0]
    eps = np.finfo(float).eps
    for X0, X1 in ((S, r["S"]), (T, r["T"])):
        A = Q @ X0 @ Z.T
        assert np.linalg.norm(A - r["Q"] @ X1 @ r["Z"].T) / np.linalg.norm(A) <= 100 * n * eps
    # the selection mask describes the blocks where they ended up: every selected row's block
    # eigenvalues are eigenvalues of the input pencil's selected blocks
    assert r["select"].sum() == r["m"]


def test_pencil_identity_T_matches_standard_path():
    # T = I, Z = Q: the pencil path reproduces the standard path's invariant subspace
    p = make_pencil(300, p2=0.25, q="householder", psel=0.35, w=64, seed=12)
    S, Q = p.np("S"), p.np("Q")
    I = np.asfortranarray(np.eye(300))
    dS, dT, dQ, dZ = _dev(S), _dev(I), _dev(Q), _dev(Q)
    r = sn.reorder_pencil(dS, dT, dQ, dZ, p.select, window=64)
    dS2, dQ2 = _dev(S), _dev(Q)
    r2 = sn.reorder(dS2, dQ2, p.select, window=64)
    torch.cuda.synchronize()
    assert r["rc"] == 0 == r2["rc"] and r["m"] == r2["m"]
    np.testing.assert_array_equal(r["bmap"], r2["bmap"])
    m = r["m"]

    def proj(X):
        q, _ = np.linalg.qr(X)
        return q @ q.T
    assert np.abs(proj(_host(dQ)[:, :m]) - proj(_host(dQ2)[:, :m])).max() <= 1e-10
    assert np.abs(_host(dT) - np.eye(300)).max() <= 1e-12


def _gpu_invariants(S0, T0, Q0, Z0, dS, dT, dQ, dZ, tol):
    """Residual and orthogonality with FP64 torch matmuls on the device (harness arithmetic;
    the dense CPU check is too slow at n = 16 384)."""
    n = S0.shape[0]
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    Qd, Zd = dQ.t(), dZ.t()                          # the tensors hold X^T
    Q0d, Z0d = torch.as_tensor(Q0).cuda(), torch.as_tensor(Z0).cuda()
    for X0, dX in ((S0, dS), (T0, dT)):
        A = Q0d @ torch.as_tensor(X0).cuda() @ Z0d.t()
        res = (torch.linalg.norm(A - Qd @ dX.t() @ Zd.t()) / torch.linalg.norm(A)).item()
        assert res <= tol, res
    for M in (Qd, Zd):
        assert torch.linalg.norm(M.t() @ M - I).item() <= tol


def test_pencil_config2_size_completes_with_prefix_parity():
    """a config-2-shaped pencil (n = 16 384, w = 256, 25 % 2x2 blocks,
    Bernoulli(0.35)) -- rejected at window 1 645 by the previous swap -- completes (rc 0) with
    the xTGEX2 two-variant re-triangularisation (G2); the first 16 windows (several DAG
    levels) match the oracle elementwise; the whole run meets the invariants."""
    p = make_pencil(16384, p2=0.25, q="householder", psel=0.35, w=256, seed=1)
    S, T, Q, Z = p.np("S"), p.np("T"), p.np("Q"), p.np("Z")
    K = 16
    dS, dT, dQ, dZ = _dev(S), _dev(T), _dev(Q), _dev(Z)
    r = sn.reorder_pencil(dS, dT, dQ, dZ, p.select, window=256, max_windows=K)
    torch.cuda.synchronize()
    ref = oracle.greorder(S, T, Q, Z, p.select, w=256, mode=1, max_windows=K, threads=os.cpu_count() or 1)
    assert r["rc"] == 0 == ref["rc"] and r["stats"]["windows"] == K == ref["stats"]["windows"]
    np.testing.assert_array_equal(r["bmap"], ref["bmap"])
    nS = np.linalg.norm(S)
    worst = 0.0
    for key, d in (("S", dS), ("T", dT), ("Q", dQ), ("Z", dZ)):
        worst = max(worst, np.abs(_host(d) - ref[key]).max() / nS)
    print("pencil n=16384 prefix K=%d levels=%d: max diff / ||S||_F = %.3g" % (K, r["stats"]["levels"], worst))
    assert worst <= 1e-9
    assert r["stats"]["levels"] >= 3
    del ref
    # the whole reordering
    dS, dT, dQ, dZ = _dev(S), _dev(T), _dev(Q), _dev(Z)
    r = sn.reorder_pencil(dS, dT, dQ, dZ, p.select, window=256)
    torch.cuda.synchronize()
    print("pencil n=16384 full: rc=%d windows=%d levels=%d swaps=%d ms_device=%.1f"
          % (r["rc"], r["stats"]["windows"], r["stats"]["levels"], r["stats"]["swaps"], r["stats"]["ms_device"]))
    assert r["rc"] == 0
    n = S.shape[0]
    b0 = blocks_of(bmap_from_S(S))
    flags = np.array([bool(p.select[q] or (sz == 2 and p.select[q + 1])) for q, sz in b0])
    sizes = np.array([sz for _, sz in b0])
    order = stable_partition(sizes, flags)
    exp_bmap = np.concatenate([[0] if sizes[t] == 1 else [1, 2] for t in order]).astype(np.int8)
    np.testing.assert_array_equal(r["bmap"], exp_bmap)
    np.testing.assert_array_equal(check_gstructure(_host(dS), _host(dT)), exp_bmap)
    _gpu_invariants(S, T, Q, Z, dS, dT, dQ, dZ, 100 * n * np.finfo(float).eps)


@pytest.mark.parametrize("n,p2,w,psel,seed,clusters", [
    (513, 0.5, 128, 0.5, 6, (2, 3, 8)), (700, 0.25, 256, 0.2, 7, (0, 4)), (2000, 0.25, 128, 0.35, 12, (0,))])
def test_pencil_cluster_split_bitwise(n, p2, w, psel, seed, clusters):
    """opts.pencil_cluster: the window task on a cluster of C CTAs (every CTA evaluates the
    step's transforms, the applications are split) gives bitwise the one-CTA result."""
    p = make_pencil(n, p2=p2, q="householder", psel=psel, w=w, seed=seed)
    _, r1 = _run(p, w, pencil_cluster=1)
    assert r1["rc"] == 0
    for c in clusters:
        _, rc = _run(p, w, pencil_cluster=c)
        assert rc["rc"] == 0
        for key in ("S", "T", "Q", "Z"):
            np.testing.assert_array_equal(rc[key], r1[key], err_msg="%s C=%d" % (key, c))
        np.testing.assert_array_equal(rc["bmap"], r1["bmap"])
        assert rc["stats"]["swaps"] == r1["stats"]["swaps"]


def test_pencil_cluster_forced_rejection_bitwise():
    p = make_pencil(400, p2=0.25, q="householder", psel=0.4, w=64, seed=11)
    _, r1 = _run(p, 64, force_reject_window=3, force_reject_swap=40, pencil_cluster=1)
    _, r4 = _run(p, 64, force_reject_window=3, force_reject_swap=40, pencil_cluster=4)
    assert r1["rc"] == 1 == r4["rc"]
    assert r1["stats"]["rejected_window"] == r4["stats"]["rejected_window"] == 3
    for key in ("S", "T", "Q", "Z"):
        np.testing.assert_array_equal(r4[key], r1[key])


def test_pencil_host_buffers_match_device_buffers():
    """Host (pageable) S, T, Q, Z are staged through device copies inside the call: bitwise the
    device-buffer result, for a padded leading dimension too (through the raw C ABI)."""
    p = make_pencil(333, p2=0.25, q="householder", psel=0.4, w=64, seed=13)
    (S, T, Q, Z), rd = _run(p, 64)
    assert rd["rc"] == 0
    hs = [torch.as_tensor(np.ascontiguousarray(X.T)) for X in (S, T, Q, Z)]   # CPU tensors
    rh = sn.reorder_pencil(*hs, p.select, window=64)
    assert rh["rc"] == 0 and rh["m"] == rd["m"]
    assert rh["stats"]["ms_h2d"] > 0 and rh["stats"]["ms_d2h"] > 0
    for key, t in zip(("S", "T", "Q", "Z"), hs):
        np.testing.assert_array_equal(t.numpy().T, rd[key], err_msg=key)
    np.testing.assert_array_equal(rh["bmap"], rd["bmap"])
    # ld = n + 3 (column-major with padding), Q absent, through the C ABI
    import ctypes as C
    n, ld = S.shape[0], S.shape[0] + 3
    pads = []
    for X in (S, T, Z):
        A = np.zeros((ld, n), order="F")
        A[:n, :] = X
        pads.append(A)
    o = sn.default_opts(window=64)
    sel = np.ascontiguousarray(p.select, np.int32).copy()
    m = C.c_int64()
    bm = np.zeros(n, np.int8)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    rc = sn.lib().sn_reorder_pencil_ex(C.byref(o), n, ptr(pads[0]), ld, ptr(pads[1]), ld, None, n, ptr(pads[2]), ld,
                                       ptr(sel), C.byref(m), ptr(bm), None, None)
    (_, _, _, _), rn = _run(p, 64, with_q=False)
    assert rc == 0 == rn["rc"]
    np.testing.assert_array_equal(pads[0][:n], rn["S"])
    np.testing.assert_array_equal(pads[1][:n], rn["T"])
    np.testing.assert_array_equal(pads[2][:n], rn["Z"])
