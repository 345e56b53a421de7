"""GPU parity of the bulge-chasing sweep (-m gpu, through the C ABI).

sn_qr_sweep (chains of bulges chased through windows, reflectors accumulated and applied by
the DMMA panel kernels) against the oracle's or_qr_sweep (bulges one after another, every
reflector applied at once; pinned to the explicit QR step and LAPACK dlaqr5 in
tests/test_oracle_sweep.py) on the same seeded Hessenberg matrices and shifts.  Reading B4:
both apply the same reflectors in exact arithmetic, in a different order (window
accumulation, chains in flight), so H and Q agree elementwise to rounding; bar 1e-9 ||H||_F
as for S and Q in the reordering, measured maxima printed.  Plus the invariants (exact
Hessenberg structure, residual, orthogonality) at the bench size.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1905_04975_b200 as sn
from tests.helpers import EPS
from workloads import make_hessenberg

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def built():
    sn.build()
    assert torch.cuda.is_available()


def _compare(h, nq=None, **opts):
    H0 = h.H_np().copy(order="F")
    Q0 = h.Q_np().copy(order="F") if h.Q is not None else None
    Hd, Qd = h.H.clone(), (h.Q.clone() if h.Q is not None else None)
    r = sn.qr_sweep(Hd, Qd, h.sr, h.si, **opts)
    torch.cuda.synchronize()
    assert r["rc"] == 0, r["rc"]
    if nq is not None and Q0 is not None:
        rows = np.sort(np.random.default_rng(1).choice(h.n, nq, replace=False))
        rc, H1, Q1 = oracle.qr_sweep(H0, np.asfortranarray(Q0[rows]), h.sr, h.si, inplace=True)
        Qg = Qd[:, torch.as_tensor(rows, device=Qd.device)].cpu().numpy().T
    else:
        rc, H1, Q1 = oracle.qr_sweep(H0, Q0, h.sr, h.si, inplace=True)
        Qg = Qd.cpu().numpy().T if Qd is not None else None
    assert rc == 0
    Hg = Hd.cpu().numpy().T
    nH = np.linalg.norm(H1)
    dH = np.abs(Hg - H1).max() / nH
    dQ = np.abs(Qg - Q1).max() if Qg is not None else 0.0
    print("n=%d shifts=%d windows=%d levels=%d: max|dH|/||H||=%.3g max|dQ|=%.3g" % (
        h.n, len(h.sr), r["stats"]["windows"], r["stats"]["levels"], dH, dQ))
    assert np.count_nonzero(np.tril(Hg, -2)) == 0
    assert dH <= TOL and dQ <= TOL
    return r


@pytest.mark.parametrize("n,ns,q,window,chain,seed", [
    (3, 2, "householder", 256, 32, 1),        # smallest: one 3-reflector and one 2-reflector
    (7, 4, "householder", 16, 2, 2),          # several tiny windows
    (64, 8, "identity", 32, 4, 3),
    (300, 16, "householder", 64, 8, 4),       # several chains, ragged last window
    (1000, 64, "householder", 256, 32, 5),    # two chains in flight
    (1500, 40, "none", 128, 12, 6),           # Q = NULL, chains of 12
    (2048, 256, "householder", 256, 32, 7),   # four chains
])
def test_sweep_matches_oracle(n, ns, q, window, chain, seed):
    h = make_hessenberg(n, ns, q=q, seed=seed, device="cuda")
    _compare(h, window=window, bulges_per_chain=chain)


def test_sweep_trailing_shifts_invariants():
    """Eigenvalue-estimate shifts (the trailing block's eigenvalues) nearly deflate the
    sweep's output, where it is ill-conditioned (LAPACK xLAQR5 and the oracle differ at
    O(1)): check backward stability only -- exact Hessenberg structure, residual,
    orthogonality, eigenvalues."""
    h = make_hessenberg(1000, 64, q="householder", seed=5, device="cuda", shifts="trailing")
    H0, Q0 = h.H_np().copy(order="F"), h.Q_np().copy(order="F")
    A = Q0 @ H0 @ Q0.T
    H, Q = h.H.clone(), h.Q.clone()
    r = sn.qr_sweep(H, Q, h.sr, h.si)
    torch.cuda.synchronize()
    assert r["rc"] == 0
    Hg, Qg = H.cpu().numpy().T, Q.cpu().numpy().T
    n = h.n
    assert np.count_nonzero(np.tril(Hg, -2)) == 0
    assert np.linalg.norm(A - Qg @ Hg @ Qg.T) / np.linalg.norm(A) <= 100 * n * EPS
    assert np.linalg.norm(Qg.T @ Qg - np.eye(n)) <= 100 * n * EPS


@pytest.mark.parametrize("window,chain", [(160, 16), (128, 12), (256, 32)])
def test_sweep_executor_variants_bitwise(window, chain):
    """The Q stream and the lookahead (critical strips first, the rest overlapping the next
    window kernel; corner order closed as in the reordering) change only the order of
    independent work: bitwise equal to the serial executor, with several chains in flight."""
    h = make_hessenberg(1500, 96, q="householder", seed=8, device="cuda")
    H1, Q1 = h.H.clone(), h.Q.clone()
    sn.qr_sweep(H1, Q1, h.sr, h.si, window=window, bulges_per_chain=chain, lookahead=0, q_stream_overlap=0)
    for kw in (dict(), dict(lookahead=0), dict(q_stream_overlap=0)):
        H2, Q2 = h.H.clone(), h.Q.clone()
        sn.qr_sweep(H2, Q2, h.sr, h.si, window=window, bulges_per_chain=chain, **kw)
        torch.cuda.synchronize()
        assert torch.equal(H1, H2) and torch.equal(Q1, Q2), kw


def test_sweep_arguments():
    h = make_hessenberg(50, 4, q="identity", seed=9, device="cuda")
    Hb = h.H.clone()
    Hb[3, 20] = 1.0                                   # H[20, 3] != 0: not Hessenberg
    assert sn.qr_sweep(Hb, None, h.sr, h.si)["rc"] == -2
    assert sn.qr_sweep(h.H.clone(), None, h.sr[:3], h.si[:3])["rc"] == -6
    assert sn.qr_sweep(h.H.clone(), None, [1.0, 2.0], [1.0, -1.0])["rc"] == -8
    assert sn.qr_sweep(h.H.clone(), None, h.sr, h.si, bulges_per_chain=64)["rc"] == sn.SN_ERR_UNSUPPORTED
    H = h.H.clone()
    assert sn.qr_sweep(H, None, [], [])["rc"] == 0 and torch.equal(H, h.H)


def test_sweep_bench_size_one_bulge_parity_and_invariants():
    """n = 40 000 (BASELINE config-3 order), Q random orthogonal: one bulge (2 shifts) against
    the full oracle sweep (all of H, a 2048-row sample of Q); then the bench's 256-shift sweep
    with its invariants: exact Hessenberg structure, the sketched residual ||(A - Q H Q^T) X||
    / ||A X|| and orthogonality (harness FP64 matmuls), <= 100 n eps."""
    h = make_hessenberg(40000, 2, q="householder", seed=1, device="cuda")
    _compare(h, nq=2048)
    h = make_hessenberg(40000, 256, q="householder", seed=1, device="cuda")
    n = h.n
    H, Q = h.H, h.Q
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.randn((n, 16), dtype=torch.float64, device="cuda", generator=g)
    AX = Q.t() @ (H.t() @ (Q @ X))
    r = sn.qr_sweep(H, Q, h.sr, h.si)
    torch.cuda.synchronize()
    assert r["rc"] == 0
    st = r["stats"]
    print("sweep n=40000 shifts=256: windows=%d levels=%d ms_device=%.1f eq TF/s=%.2f" % (
        st["windows"], st["levels"], st["ms_device"], st["eq_flops"] / st["ms_device"] / 1e9))
    assert not bool((torch.triu(H, 2) != 0).any().item())   # H[i, j] = Ht[j, i] = 0 for i >= j + 2
    res = torch.linalg.norm(Q.t() @ (H.t() @ (Q @ X)) - AX).item() / torch.linalg.norm(AX).item()
    orth = torch.linalg.norm(Q @ (Q.t() @ X) - X).item() / torch.linalg.norm(X).item()
    print("residual %.3g orthogonality %.3g" % (res, orth))
    assert res <= 100 * n * EPS and orth <= 100 * n * EPS
