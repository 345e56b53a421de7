"""The sharded data path on one GPU (-m gpu): sn_reorder_schur_dist_local runs P ranks'
shards on cuda:0 with the same program, kernels and halo/straddle logic as the NCCL path
(messages become device copies).  Bar: block map and selection bit-exact, S and Q within
1e-9 ||S||_F of the oracle (BASELINE north_star), and bitwise equal to the one-GPU path
(every output element is accumulated over K in the same order by the same kernels).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1905_04975_b200 as sn
from tests.helpers import check_reordering
from workloads import make_problem

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def built():
    sn.build()
    assert torch.cuda.is_available()


def run_dist(p, P, bc, w, q=True, **opts):
    S = p.S.cuda()
    Q = p.Q.cuda() if (q and p.Q is not None) else None
    shards = [sn.shard(S, Q, P, bc, r) for r in range(P)]
    Sl = [s for s, _ in shards]
    Ql = None if Q is None else [x for _, x in shards]
    got = sn.reorder_dist_local(Sl, Ql, p.select, p.n, bc, window=w, validate_lower=1, **opts)
    torch.cuda.synchronize()
    Sg, Qg = sn.unshard(Sl, Ql, p.n, P, bc)
    return got, Sg, Qg


def run_single(p, w, q=True, **opts):
    S = p.S.cuda().contiguous()
    Q = p.Q.cuda().contiguous() if (q and p.Q is not None) else None
    got = sn.reorder(S, Q, p.select, window=w, **opts)
    torch.cuda.synchronize()
    return got, S.cpu().numpy().T, (None if Q is None else Q.cpu().numpy().T)


@pytest.mark.parametrize("n,w,bc,P,seed", [
    (700, 64, 64, 1, 1), (700, 64, 64, 2, 2), (900, 64, 128, 3, 3), (1000, 128, 128, 4, 4),
    (1200, 256, 256, 2, 5), (1500, 128, 512, 3, 6), (640, 32, 32, 8, 7)])
def test_dist_local_parity(n, w, bc, P, seed):
    p = make_problem(n, 0.25, "householder", "bernoulli", 0.35, w, seed=seed)
    S0, Q0 = p.S_np().copy(order="F"), p.Q_np().copy(order="F")
    ref = oracle.reorder(S0, Q0, p.select, w=w, mode=1)
    got, Sg, Qg = run_dist(p, P, bc, w)
    assert got["rc"] == 0 == ref["rc"]
    assert got["m"] == ref["m"]
    np.testing.assert_array_equal(got["bmap"], ref["bmap"])
    np.testing.assert_array_equal(got["select"], ref["select"])
    nS = np.linalg.norm(S0)
    dS, dQ = np.abs(Sg - ref["S"]).max(), np.abs(Qg - ref["Q"]).max()
    print("P=%d bc=%d max|dS|/||S||=%.3g max|dQ|=%.3g" % (P, bc, dS / nS, dQ))
    assert dS <= TOL * nS and dQ <= TOL * nS
    assert got["stats"]["windows"] == ref["stats"]["windows"]
    check_reordering(S0, Q0, p.select, Sg, Qg, got["select"], got["m"], got["bmap"])
    # same kernels, same K order per element: bitwise equal to the one-GPU executor
    g1, S1, Q1 = run_single(p, w)
    assert np.array_equal(S1, Sg) and np.array_equal(Q1, Qg)


def test_dist_local_worst_case_chain():
    p = make_problem(1024, 0.5, "householder", "trailing_half", None, 128, seed=8)
    S0, Q0 = p.S_np().copy(order="F"), p.Q_np().copy(order="F")
    ref = oracle.reorder(S0, Q0, p.select, w=128, mode=1)
    got, Sg, Qg = run_dist(p, 4, 128, 128)
    assert got["rc"] == 0
    np.testing.assert_array_equal(got["bmap"], ref["bmap"])
    nS = np.linalg.norm(S0)
    assert np.abs(Sg - ref["S"]).max() <= TOL * nS and np.abs(Qg - ref["Q"]).max() <= TOL * nS


def test_dist_local_without_Q_and_trivial():
    p = make_problem(600, 0.25, "householder", "bernoulli", 0.35, 64, seed=9)
    got, Sg, _ = run_dist(p, 3, 64, 64, q=False)
    g1, S1, _ = run_single(p, 64, q=False)
    assert got["rc"] == 0 and np.array_equal(S1, Sg)
    # nothing selected: bitwise no-op
    p2 = make_problem(300, 0.25, "identity", "none", None, 32, seed=10)
    got, Sg, Qg = run_dist(p2, 2, 32, 32)
    assert got["rc"] == 0 and got["m"] == 0
    assert np.array_equal(Sg, p2.S_np()) and np.array_equal(Qg, p2.Q_np())


def test_dist_local_forced_rejection_consistent_state():
    """A rejected swap stops the sharded run at a valid, partially reordered Schur form;
    which other windows of the rejecting level completed may differ from the one-GPU run
    (they are independent), so the checks are the invariants, not equality."""
    from tests.helpers import EPS, bmap_from_S
    p = make_problem(800, 0.25, "householder", "bernoulli", 0.35, 64, seed=12)
    got, Sg, Qg = run_dist(p, 3, 64, 64, force_reject_window=9, force_reject_swap=7)
    assert got["rc"] == sn.SN_ERR_REJECTED
    assert got["stats"]["rejected_window"] == 9
    n = p.n
    S0, Q0 = p.S_np(), p.Q_np()
    A = Q0 @ S0 @ Q0.T
    assert np.linalg.norm(A - Qg @ Sg @ Qg.T) / np.linalg.norm(A) <= 100 * n * EPS
    assert np.linalg.norm(Qg.T @ Qg - np.eye(n)) <= 100 * n * EPS
    np.testing.assert_array_equal(got["bmap"], bmap_from_S(Sg))
    assert int(got["select"].sum()) == got["m"]
    row, n1 = got["stats"]["rejected_row"], got["stats"]["rejected_n1"]
    assert got["select"][row + n1] == 1 and got["select"][row] == 0


def test_dist_nccl_world1_matches_single():
    """The NCCL entry point (sn_dist_init + sn_reorder_schur_dist) with a one-rank
    communicator: every collective of the sharded program is issued (1-rank broadcast and
    all-reduce) and the straddle messages become local copies; bitwise equal to one GPU."""
    p = make_problem(900, 0.25, "householder", "bernoulli", 0.35, 64, seed=13)
    sn.dist_init(0, 1, 0, broadcast_id=lambda b: b)
    try:
        Sl, Ql = sn.shard(p.S.cuda(), p.Q.cuda(), 1, 64, 0)
        got = sn.reorder_dist(Sl, Ql, p.select, p.n, 64, window=64)
        torch.cuda.synchronize()
        assert got["rc"] == 0, got["rc"]
        Sg, Qg = sn.unshard([Sl], [Ql], p.n, 1, 64)
        g1, S1, Q1 = run_single(p, 64)
        assert np.array_equal(S1, Sg) and np.array_equal(Q1, Qg)
        np.testing.assert_array_equal(got["bmap"], g1["bmap"])
        # host shards (staged inside the call)
        Sh, Qh = sn.shard(p.S, p.Q, 1, 64, 0)
        got = sn.reorder_dist(Sh, Qh, p.select, p.n, 64, window=64)
        assert got["rc"] == 0
        Sg2, Qg2 = sn.unshard([Sh], [Qh], p.n, 1, 64)
        assert np.array_equal(S1, Sg2) and np.array_equal(Q1, Qg2)
    finally:
        sn.dist_finalize()


def test_dist_local_config3_fullsize_bitwise():
    """The sharded program at the bench size (config 3, n = 40 000, bc = 512) for 4 ranks on
    one device: S and Q bitwise equal to the one-GPU executor (compared on the device)."""
    from workloads import make_config
    p = make_config(3, seed=1, device="cuda")
    n, P, bc = p.n, 4, 512
    shards = [sn.shard(p.S, p.Q, P, bc, r) for r in range(P)]
    Sl = [s for s, _ in shards]
    Ql = [q for _, q in shards]
    del shards
    g1 = sn.reorder(p.S, p.Q, p.select, window=p.w)
    got = sn.reorder_dist_local(Sl, Ql, p.select, n, bc, window=p.w)
    torch.cuda.synchronize()
    assert g1["rc"] == 0 and got["rc"] == 0
    np.testing.assert_array_equal(got["bmap"], g1["bmap"])
    assert got["stats"]["windows"] == g1["stats"]["windows"]
    for r in range(P):
        cols = torch.as_tensor(sn.owned_columns(n, P, bc, r), device="cuda")
        assert torch.equal(p.S[cols], Sl[r][:len(cols)])
        _, q0, q1 = sn.dist_layout(n, P, bc, r)
        assert torch.equal(p.Q[:, q0:q1], Ql[r][:, :q1 - q0])
