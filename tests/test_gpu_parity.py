"""Parity of the CUDA path (through the C ABI) with the CPU oracle, on the GPU (-m gpu).

Bar (BASELINE.json north_star): block map and selection mask bit-exact; S and Q elementwise
within 1e-9 * ||S||_F; the invariants of tests/helpers.check_reordering.  The GPU executes
the swaps of a window in a different (commuting) order than the oracle (inner windows,
DESIGN.md §4), so agreement is to rounding, far inside the bar; the measured maxima are
printed.  Inputs come from workloads/ only; expected values only from oracle/.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import paper_1905_04975_b200 as sn
from tests.helpers import EPS, bmap_from_S, blocks_of, check_reordering
from workloads import make_config, make_problem

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def built():
    sn.build()
    assert torch.cuda.is_available()


def run_both(p, w=None, q=True, oracle_threads=0, **opts):
    w = w or p.w
    S0 = p.S_np().copy(order="F")
    Q0 = p.Q_np().copy(order="F") if (q and p.Q is not None) else None
    if oracle_threads:
        # the oracle's panel rows / columns on the host's cores: bitwise the one-thread result
        # (tests/test_oracle_pins.py), minutes less of the GPU suite at n = 4096
        ref = oracle.reorder_threads(S0, Q0, p.select, w, oracle_threads)
    else:
        ref = oracle.reorder(S0, Q0, p.select, w=w, mode=1)
    S = p.S.cuda().contiguous()
    Q = p.Q.cuda().contiguous() if Q0 is not None else None
    got = sn.reorder(S, Q, p.select, window=w, validate_lower=1, **opts)
    torch.cuda.synchronize()
    return S0, Q0, ref, got, S.cpu().numpy().T, (Q.cpu().numpy().T if Q is not None else None)


def assert_parity(S0, Q0, ref, got, Sg, Qg, label=""):
    assert got["rc"] == 0 == ref["rc"]
    assert got["m"] == ref["m"]
    np.testing.assert_array_equal(got["bmap"], ref["bmap"])
    np.testing.assert_array_equal(got["select"], ref["select"])
    nS = np.linalg.norm(S0)
    dS = np.abs(Sg - ref["S"]).max() if S0.size else 0.0
    dQ = np.abs(Qg - ref["Q"]).max() if Qg is not None and Qg.size else 0.0
    print("%s max|dS|/||S||=%.3g max|dQ|=%.3g windows=%d swaps=%d" % (
        label, dS / max(nS, 1e-300), dQ, got["stats"]["windows"], got["stats"]["swaps"]))
    assert dS <= TOL * nS and dQ <= TOL * nS
    assert got["stats"]["windows"] == ref["stats"]["windows"]
    assert got["stats"]["swaps"] == ref["stats"]["swaps"]
    return dS / max(nS, 1e-300), dQ


def test_config0_parity():
    p = make_config(0, seed=1)
    S0, Q0, ref, got, Sg, Qg = run_both(p)
    assert_parity(S0, Q0, ref, got, Sg, Qg, "config0")
    check_reordering(S0, Q0, p.select, Sg, Qg, got["select"], got["m"], got["bmap"])


@pytest.mark.parametrize("n,p2,w,psel,q,seed", [
    (97, 0.25, 16, 0.5, "householder", 3),      # ragged: n not a multiple of any tile
    (300, 0.5, 32, 0.35, "householder", 4),
    (511, 0.0, 64, 0.6, "householder", 5),      # all 1x1 (Givens only)
    (640, 100.0, 64, 0.3, "householder", 6),    # all 2x2 (Householder only)
    (700, 0.25, 128, 0.35, "identity", 7),
    (1000, 0.25, 256, 0.35, "householder", 8),  # several 256-row windows, ragged tails
    (1200, 0.5, 200, 0.5, "none", 9),           # Q = NULL, w not a power of two
    (64, 0.25, 4, 0.5, "householder", 10),      # smallest window
    (130, 0.25, 5, 0.5, "householder", 11),     # odd window
])
def test_random_parity(n, p2, w, psel, q, seed):
    p = make_problem(n, p2=p2, q=q, psel=psel, w=w, seed=seed)
    S0, Q0, ref, got, Sg, Qg = run_both(p)
    assert_parity(S0, Q0, ref, got, Sg, Qg, "n=%d w=%d" % (n, w))
    check_reordering(S0, Q0, p.select, Sg, Qg, got["select"], got["m"], got["bmap"])


def test_config1_parity():
    """BASELINE config 1 (n = 4096, w = 128, random orthogonal Q), full oracle run."""
    p = make_config(1, seed=1, device="cuda")
    p.S = p.S.cpu(); p.Q = p.Q.cpu()
    S0, Q0, ref, got, Sg, Qg = run_both(p, oracle_threads=os.cpu_count() or 1)
    assert_parity(S0, Q0, ref, got, Sg, Qg, "config1")
    check_reordering(S0, Q0, p.select, Sg, Qg, got["select"], got["m"], got["bmap"])


def test_block_diagonal_exact():
    """Zero coupling: every transform is a signed (block) permutation, so the GPU result is
    exact -- |entries| equal to the oracle's bitwise."""
    p = make_problem(300, p2=0.25, q="householder", psel=0.4, w=32, seed=12)
    S = p.S_np().copy(order="F")
    bm = bmap_from_S(S)
    mask = np.zeros_like(S, bool)
    for r, sz in blocks_of(bm):
        mask[r:r + sz, r:r + sz] = True
    S[~mask] = 0.0
    p.S = torch.from_numpy(np.ascontiguousarray(S.T))
    S0, Q0, ref, got, Sg, Qg = run_both(p)
    # signed, bitwise: both sides build the same signed permutations from
    # exact data (f = 0 Givens, tau = 1 reflectors, standard blocks unchanged by xLANV2)
    assert np.array_equal(Sg, ref["S"])
    assert np.array_equal(Qg, ref["Q"])
    np.testing.assert_array_equal(got["bmap"], ref["bmap"])
    # and S is an exact signed block permutation of the input
    off = Sg.copy()
    for r, sz in blocks_of(got["bmap"]):
        off[r:r + sz, r:r + sz] = 0.0
    assert np.count_nonzero(off) == 0


def test_trivial_selections_bitwise_noop():
    p = make_problem(500, q="householder", sel="all", w=64, seed=13)
    for sel in (p.select, np.zeros_like(p.select)):
        S = p.S.cuda(); Q = p.Q.cuda()
        got = sn.reorder(S, Q, sel, window=64)
        assert got["rc"] == 0 and got["stats"]["windows"] == 0
        assert torch.equal(S.cpu(), p.S) and torch.equal(Q.cpu(), p.Q)


def test_idempotent_second_call():
    p = make_problem(800, q="householder", psel=0.35, w=128, seed=14)
    S = p.S.cuda(); Q = p.Q.cuda()
    r1 = sn.reorder(S, Q, p.select, window=128)
    S1, Q1 = S.clone(), Q.clone()
    r2 = sn.reorder(S, Q, r1["select"], window=128)
    assert r2["rc"] == 0 and r2["stats"]["windows"] == 0
    assert torch.equal(S, S1) and torch.equal(Q, Q1)


def test_host_pointer_path_matches_device_path():
    p = make_problem(777, q="householder", psel=0.35, w=128, seed=15)
    Sd, Qd = p.S.cuda(), p.Q.cuda()
    rd = sn.reorder(Sd, Qd, p.select, window=128)
    Sh, Qh = p.S.clone(), p.Q.clone()
    rh = sn.reorder(Sh, Qh, p.select, window=128)
    assert rd["rc"] == rh["rc"] == 0
    assert torch.equal(Sd.cpu(), Sh) and torch.equal(Qd.cpu(), Qh)
    assert rh["stats"]["ms_h2d"] > 0


def test_plain_abi_signature():
    """sn_reorder_schur(n, S, ldS, Q, ldQ, select, &m) with raw device pointers."""
    p = make_problem(256, q="householder", psel=0.5, w=64, seed=16)
    S, Q = p.S.cuda(), p.Q.cuda()
    sel = p.select.astype(np.int32).copy()
    rc, m = sn.sn_reorder_schur(256, S.data_ptr(), 256, Q.data_ptr(), 256, sel)
    torch.cuda.synchronize()
    assert rc == 0 and m == int(p.select.sum())
    check_reordering(p.S_np(), p.Q_np(), p.select, S.cpu().numpy().T, Q.cpu().numpy().T, sel, m,
                     bmap_from_S(S.cpu().numpy().T))


def test_edge_sizes():
    for n in (1, 2, 3):
        p = make_problem(n, p2=0.5, q="householder", psel=0.5, w=4, seed=17 + n)
        S0, Q0, ref, got, Sg, Qg = run_both(p)
        assert_parity(S0, Q0, ref, got, Sg, Qg, "n=%d" % n)


def test_not_quasi_triangular_rejected():
    p = make_problem(50, q="identity", psel=0.5, w=8, seed=20)
    S = p.S.clone()
    S[3, 10] = 1.0            # S[10, 3] != 0: below the subdiagonal
    r = sn.reorder(S.cuda(), p.Q.cuda(), p.select, window=8, validate_lower=1)
    assert r["rc"] == -2
    S = p.S.clone()
    S[4, 5] = 1.0; S[5, 6] = 1.0   # consecutive nonzero subdiagonal entries
    r = sn.reorder(S.cuda(), p.Q.cuda(), p.select, window=8)
    assert r["rc"] == -2


def test_forced_rejection_consistent_state():
    p = make_problem(600, p2=0.25, q="householder", psel=0.4, w=64, seed=21)
    S, Q = p.S.cuda(), p.Q.cuda()
    sch_full = sn.reorder(p.S.cuda(), p.Q.cuda(), p.select, window=64)
    t = sch_full["stats"]["windows"] // 2
    r = sn.reorder(S, Q, p.select, window=64, force_reject_window=t, force_reject_swap=3)
    assert r["rc"] == sn.SN_ERR_REJECTED
    assert r["stats"]["rejected_window"] == t
    Sg, Qg = S.cpu().numpy().T, Q.cpu().numpy().T
    n = p.n
    A = p.Q_np() @ p.S_np() @ p.Q_np().T
    assert np.linalg.norm(A - Qg @ Sg @ Qg.T) / np.linalg.norm(A) <= 100 * n * EPS
    assert np.linalg.norm(Qg.T @ Qg - np.eye(n)) <= 100 * n * EPS
    np.testing.assert_array_equal(r["bmap"], bmap_from_S(Sg))
    assert int(r["select"].sum()) == r["m"]
    row, n1 = r["stats"]["rejected_row"], r["stats"]["rejected_n1"]
    assert r["select"][row + n1] == 1 and r["select"][row] == 0


def test_prefix_parity_config2():
    """BASELINE config 2 (n = 16384, w = 256): the first windows of the schedule on GPU and
    oracle (SURVEY c5 'prefix parity'), compared over all of S and Q."""
    p = make_config(2, seed=1, device="cuda")
    K = 6
    S0 = np.asfortranarray(p.S.cpu().numpy().T)
    Q0 = np.asfortranarray(p.Q.cpu().numpy().T)
    S, Q = p.S.clone(), p.Q.clone()
    got = sn.reorder(S, Q, p.select, window=p.w, max_windows=K)
    ref = oracle.reorder_threads(S0, Q0, p.select, p.w, os.cpu_count() or 1, max_windows=K)
    assert got["rc"] == 0 == ref["rc"]
    assert got["stats"]["windows"] == ref["stats"]["windows"] == K
    np.testing.assert_array_equal(got["bmap"], ref["bmap"])
    nS = np.linalg.norm(S0)
    dS = np.abs(S.cpu().numpy().T - ref["S"]).max()
    dQ = np.abs(Q.cpu().numpy().T - ref["Q"]).max()
    print("config2 prefix K=%d: max|dS|/||S||=%.3g max|dQ|=%.3g" % (K, dS / nS, dQ))
    assert dS <= TOL * nS and dQ <= TOL * nS


@pytest.mark.parametrize("opts", [dict(lookahead=0), dict(q_stream_overlap=0), dict(serialize=1),
                                  dict(lookahead=0, q_stream_overlap=0, serialize=1), dict(inner_window=32),
                                  dict(inner_window=16, lookahead=1)])
def test_executor_variants_parity(opts):
    """Every executor configuration (streams, lookahead, inner window size) meets the bar."""
    p = make_problem(1500, p2=0.25, q="householder", psel=0.35, w=256, seed=30)
    S0, Q0, ref, got, Sg, Qg = run_both(p, **opts)
    assert_parity(S0, Q0, ref, got, Sg, Qg, str(opts))


@pytest.mark.parametrize("pad", [1, 3])
def test_padded_leading_dimension(pad):
    """ldS = ldQ = n + pad (odd: the 8-byte copy paths; the buffers carry garbage padding)."""
    p = make_problem(777, q="householder", psel=0.35, w=256, seed=31)
    n, ld = p.n, p.n + pad
    S0, Q0 = p.S_np().copy(order="F"), p.Q_np().copy(order="F")
    ref = oracle.reorder(S0, Q0, p.select, w=256, mode=1)
    Sb = torch.full((n, ld), float("nan"), dtype=torch.float64)
    Qb = torch.full((n, ld), float("nan"), dtype=torch.float64)
    Sb[:, :n] = p.S; Qb[:, :n] = p.Q
    Sb, Qb = Sb.cuda(), Qb.cuda()
    sel = p.select.astype(np.int32).copy()
    rc, m = sn.sn_reorder_schur(n, Sb.data_ptr(), ld, Qb.data_ptr(), ld, sel)
    torch.cuda.synchronize()
    assert rc == 0 and m == ref["m"]
    Sg, Qg = Sb[:, :n].cpu().numpy().T, Qb[:, :n].cpu().numpy().T
    assert torch.isnan(Sb[:, n:]).all() and torch.isnan(Qb[:, n:]).all()
    nS = np.linalg.norm(S0)
    assert np.abs(Sg - ref["S"]).max() <= TOL * nS and np.abs(Qg - ref["Q"]).max() <= TOL * nS
    np.testing.assert_array_equal(sel, ref["select"])


def _eig_keys(S, bmap):
    """Per block (row, size): its eigenvalue key (1x1: the diagonal entry; 2x2: the complex
    pair's real part and |imag|, rounded) -- identifies a block across reorderings."""
    out = []
    for r, sz in blocks_of(bmap):
        if sz == 1:
            out.append((r, sz, (float(S[r, r]), 0.0)))
        else:
            e = np.linalg.eigvals(S[r:r + 2, r:r + 2])
            out.append((r, sz, (round(float(e[0].real), 8), round(abs(float(e[0].imag)), 8))))
    return out


def test_forced_rejection_two_windows_one_level():
    """several windows of one DAG level reject.  Every partial window keeps its
    own record, so the returned block map and selection describe S exactly (each block's
    eigenvalue sits where the mask says), the form is valid, and the outcome does not depend
    on CTA scheduling (two runs are bitwise equal)."""
    p = make_problem(1400, p2=0.25, q="householder", psel=0.4, w=64, seed=22)
    bm0 = bmap_from_S(p.S_np())
    sel0 = np.zeros(p.n, np.int8)
    for r, sz in blocks_of(bm0):
        sel0[r:r + sz] = 1 if p.select[r:r + sz].any() else 0
    sch = sn.schedule(bm0, sel0, 64)
    lev, cnt = np.unique(sch["level"], return_counts=True)
    target = int(lev[np.argmax(cnt)])
    assert cnt.max() >= 2, "need a level with two windows"
    outs = []
    for rep in range(2):
        S, Q = p.S.cuda(), p.Q.cuda()
        r = sn.reorder(S, Q, p.select, window=64, force_reject_window=-2 - target, force_reject_swap=2)
        torch.cuda.synchronize()
        outs.append((r, S.cpu(), Q.cpu()))
    r, St, Qt = outs[0]
    assert r["rc"] == sn.SN_ERR_REJECTED
    assert torch.equal(St, outs[1][1]) and torch.equal(Qt, outs[1][2])
    np.testing.assert_array_equal(r["bmap"], outs[1][0]["bmap"])
    assert r["stats"]["swaps"] == outs[1][0]["stats"]["swaps"]
    Sg, Qg = St.numpy().T, Qt.numpy().T
    n = p.n
    A = p.Q_np() @ p.S_np() @ p.Q_np().T
    assert np.linalg.norm(A - Qg @ Sg @ Qg.T) / np.linalg.norm(A) <= 100 * n * EPS
    assert np.linalg.norm(Qg.T @ Qg - np.eye(n)) <= 100 * n * EPS
    np.testing.assert_array_equal(r["bmap"], bmap_from_S(Sg))
    # the selection flag of every block of the output is that of its input block
    sel_of = {key: int(sel0[r0]) for r0, sz, key in _eig_keys(p.S_np(), bm0)}
    for r1, sz, key in _eig_keys(Sg, r["bmap"]):
        assert r["select"][r1] == sel_of[key], (r1, sz, key)
    assert int(r["select"].sum()) == r["m"]
    nrej = int((sch["level"] == target).sum())
    print("level %d with %d windows rejected; windows executed %d of %d" %
          (target, nrej, r["stats"]["windows"], len(sch["level"])))


def test_repeat_run_bitwise_deterministic():
    """SURVEY c5 'Determinism': a fixed stream layout gives bitwise identical results."""
    p = make_problem(2000, p2=0.25, q="householder", psel=0.35, w=256, seed=32)
    res = []
    for _ in range(3):
        S, Q = p.S.cuda(), p.Q.cuda()
        r = sn.reorder(S, Q, p.select, window=256)
        torch.cuda.synchronize()
        res.append((S.cpu(), Q.cpu(), r["bmap"]))
    for S, Q, bm in res[1:]:
        assert torch.equal(S, res[0][0]) and torch.equal(Q, res[0][1])
        np.testing.assert_array_equal(bm, res[0][2])


@pytest.mark.parametrize("opts", [dict(serialize=1, lookahead=0, q_stream_overlap=0), dict(lookahead=0),
                                  dict(q_stream_overlap=0), dict(serialize=1)])
def test_serialised_equals_pipelined_bitwise(opts):
    """The executor's concurrency (lookahead strips, Q stream, no host syncs) changes only the
    order of independent strips, never an arithmetic sequence: bitwise equal to the fully
    serialised run (SURVEY §5 asks for <= 1e-13)."""
    p = make_problem(1800, p2=0.25, q="householder", psel=0.35, w=256, seed=33)
    S1, Q1 = p.S.cuda(), p.Q.cuda()
    r1 = sn.reorder(S1, Q1, p.select, window=256)
    S2, Q2 = p.S.cuda(), p.Q.cuda()
    r2 = sn.reorder(S2, Q2, p.select, window=256, **opts)
    torch.cuda.synchronize()
    assert r1["rc"] == r2["rc"] == 0
    assert torch.equal(S1, S2) and torch.equal(Q1, Q2)


def test_natural_rejection_matches_oracle():
    """No forcing: an ill-conditioned 2x2|2x2 pair that LAPACK dtrsen and the oracle reject
    (tests/test_oracle_pins.py) is rejected by the GPU at the same pair, with the same
    partial block map and the partial S, Q within the bar; and a 2x1 pair whose moved 2x2
    block would split (reading R6) likewise."""
    from tests.test_oracle_pins import _near_pair
    from scipy.linalg import lapack
    for n1, n2, want in ((2, 2, 1), (2, 1, 2)):
        rng = np.random.default_rng(77 + n2)
        for _ in range(500):
            B = _near_pair(rng, n1, n2)
            oracle.swap(B, 0, n1, n2)
            if oracle.swap_last_reject() == want:
                break
        assert oracle.swap_last_reject() == want
        n = 5 + n1 + n2
        S = np.triu(rng.standard_normal((n, n)))
        for i, v in enumerate((4.0, -3.0, 6.5, 8.25, -7.5)):
            S[i, i] = v
        S[5:, 5:] = B
        Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
        sel = np.zeros(n, np.int32)
        sel[5 + n1:] = 1
        sel[1] = 1
        ref = oracle.reorder(np.asfortranarray(S), np.asfortranarray(Q), sel, w=8, mode=1)
        assert ref["rc"] == 1
        St = torch.from_numpy(np.ascontiguousarray(S.T)).cuda()
        Qt = torch.from_numpy(np.ascontiguousarray(Q.T)).cuda()
        got = sn.reorder(St, Qt, sel, window=8)
        torch.cuda.synchronize()
        assert got["rc"] == sn.SN_ERR_REJECTED
        assert got["stats"]["rejected_row"] == ref["stats"]["rejected_row"] == 5
        np.testing.assert_array_equal(got["bmap"], ref["bmap"])
        np.testing.assert_array_equal(got["select"], ref["select"])
        nS = np.linalg.norm(S)
        assert np.abs(St.cpu().numpy().T - ref["S"]).max() <= TOL * nS
        assert np.abs(Qt.cpu().numpy().T - ref["Q"]).max() <= TOL * nS


@pytest.mark.parametrize("n,w,opts", [(2500, 256, {}), (1500, 64, {}), (1300, 128, {}),
                                      (2200, 256, dict(q_stream_overlap=0)),
                                      (2200, 256, dict(lookahead=0, serialize=1))])
def test_fused_chain_q_bitwise(n, w, opts):
    """Row f1, fused chain updates (opts.fuse_chain): the Q updates of consecutive
    windows of a chain applied in one CTA pass per Q strip give bitwise the unfused result
    (each pass is the same arithmetic sequence; the fusion changes only when and where)."""
    p = make_problem(n, p2=0.25, q="householder", psel=0.35, w=w, seed=40 + n % 7)
    outs = []
    for fuse in (0, 1):
        S, Q = p.S.cuda(), p.Q.cuda()
        r = sn.reorder(S, Q, p.select, window=w, fuse_chain=fuse, **opts)
        torch.cuda.synchronize()
        outs.append((r, S.cpu(), Q.cpu()))
    (r0, S0, Q0), (r1, S1, Q1) = outs
    assert r0["rc"] == r1["rc"] == 0
    assert r0["stats"]["fused_q_pairs"] == 0 and r1["stats"]["fused_q_pairs"] > 0
    print("n=%d w=%d %s: %d fused pairs of %d windows" % (n, w, opts, r1["stats"]["fused_q_pairs"],
                                                         r1["stats"]["windows"]))
    assert torch.equal(S0, S1) and torch.equal(Q0, Q1)
    np.testing.assert_array_equal(r0["bmap"], r1["bmap"])


def test_fused_chain_q_oracle_parity():
    """The fused executor against the oracle (the bar of the unfused path)."""
    p = make_problem(1700, p2=0.25, q="householder", psel=0.35, w=256, seed=41)
    S0, Q0, ref, got, Sg, Qg = run_both(p, fuse_chain=1)
    assert got["stats"]["fused_q_pairs"] > 0
    assert_parity(S0, Q0, ref, got, Sg, Qg, "fuse_chain")


def test_fused_chain_q_forced_rejection():
    """A rejection inside a fused pair's levels: the predecessor's Q pass still runs when its
    successor is skipped, so the state equals the unfused run's bitwise."""
    p = make_problem(1400, p2=0.25, q="householder", psel=0.4, w=64, seed=22)
    sch = sn.reorder(p.S.cuda(), p.Q.cuda(), p.select, window=64, fuse_chain=1)
    assert sch["stats"]["fused_q_pairs"] > 0
    outs = []
    for t in (sch["stats"]["windows"] // 3, sch["stats"]["windows"] // 2):
        for fuse in (0, 1):
            S, Q = p.S.cuda(), p.Q.cuda()
            r = sn.reorder(S, Q, p.select, window=64, fuse_chain=fuse, force_reject_window=t,
                           force_reject_swap=1)
            torch.cuda.synchronize()
            assert r["rc"] == sn.SN_ERR_REJECTED
            outs.append((r, S.cpu(), Q.cpu()))
        (ra, Sa, Qa), (rb, Sb, Qb) = outs[-2:]
        assert torch.equal(Sa, Sb) and torch.equal(Qa, Qb)
        np.testing.assert_array_equal(ra["bmap"], rb["bmap"])
