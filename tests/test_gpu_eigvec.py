"""GPU parity of the eigenvector path (-m gpu, through the C ABI).

sn_eigenvectors (blocked back substitution with overflow protection + DMMA update and
back-transform GEMMs) against the oracle's or_eigvec (pinned to LAPACK xTREVC3 in
tests/test_oracle_eigvec.py) on the same seeded Schur forms.  Both normalise every vector
(pair) to max(|re| + |im|) = 1 (E5), which removes the power-of-two protection scalings, so
the columns compare elementwise; they differ by the summation order of the blocked updates
(rounding times the vectors' condition).  Bar: 1e-9 elementwise (the north star's bar for
S and Q), measured maxima printed.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_1905_04975_b200 as sn
from tests.helpers import blocks_of, bmap_from_S
from workloads import make_config, make_problem

pytestmark = pytest.mark.gpu
TOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def built():
    sn.build()
    assert torch.cuda.is_available()


def _dev(M):
    return torch.as_tensor(np.ascontiguousarray(M.T)).cuda()


def _run(S, Q, sel):
    r = sn.eigenvectors(_dev(S), None if Q is None else _dev(Q), sel, scale_exp=True)
    torch.cuda.synchronize()
    assert r["rc"] == 0, r["rc"]
    return r, r["X"].cpu().numpy().T


@pytest.mark.parametrize("n,p2,frac,q,seed", [
    (40, 0.25, 1.0, False, 1), (129, 0.5, 1.0, True, 2), (257, 0.25, 0.4, True, 3), (300, 1e9, 0.5, False, 4),
    (1000, 0.25, 0.35, True, 5), (1537, 0.0, 0.2, True, 6)])
def test_eigvec_matches_oracle(n, p2, frac, q, seed):
    p = make_problem(n, p2=p2, q="householder", psel=0.5, w=16, seed=seed)
    S = p.S_np().copy(order="F")
    Q = p.Q_np().copy(order="F") if q else None
    sel = (np.random.default_rng(seed).random(n) < frac).astype(np.int32)
    rc, Xo, eo = oracle.eigvec(S, Q, sel)
    r, Xg = _run(S, Q, sel)
    assert r["ncols"] == Xo.shape[1]
    d = np.abs(Xg - Xo).max()
    print("n=%d cols=%d max|dX|=%.3g rescales=%d" % (n, r["ncols"], d, r["stats"]["rescales"]))
    assert d <= TOL


def test_eigvec_2x2_blocks_across_tile_boundaries():
    """2x2 blocks at rows (127, 128), (255, 256): the row tiles move their boundary by one row
    so no block is split; every vector still matches."""
    rng = np.random.default_rng(11)
    n = 400
    S = np.triu(rng.standard_normal((n, n)))
    S[np.arange(n), np.arange(n)] = rng.uniform(-10, 10, n)
    for r in (127, 255, 383):
        a = rng.uniform(-10, 10)
        S[r, r] = S[r + 1, r + 1] = a
        S[r, r + 1] = rng.uniform(0.5, 3)
        S[r + 1, r] = -rng.uniform(0.5, 3)
        S[r + 1, r + 2:] = S[r + 1, r + 2:]   # upper part kept
    S = np.asfortranarray(S)
    assert (bmap_from_S(S)[[127, 128, 255, 256]] == [1, 2, 1, 2]).all()
    sel = np.ones(n, np.int32)
    rc, Xo, _ = oracle.eigvec(S, None, sel)
    r, Xg = _run(S, None, sel)
    assert np.abs(Xg - Xo).max() <= TOL


@pytest.mark.parametrize("big,n", [(1e300, 8), (1e30, 300)])
def test_eigvec_overflow_protection(big, n):
    """Entries that overflow an unprotected back substitution (SPEC eigvec example): finite
    output, protective rescalings recorded, equal to the oracle after normalisation."""
    rng = np.random.default_rng(3)
    S = np.asfortranarray(np.triu(np.full((n, n), big), 1) + np.diag(rng.uniform(-1, 1, n)))
    sel = np.ones(n, np.int32)
    rc, Xo, eo = oracle.eigvec(S, None, sel)
    r, Xg = _run(S, None, sel)
    assert np.isfinite(Xg).all()
    assert r["stats"]["rescales"] > 0 and r["scale_exp"].max() > 0
    print("big=%g: rescales=%d max e=%d (oracle %d) max|dX|=%.3g" % (
        big, r["stats"]["rescales"], r["scale_exp"].max(), eo.max(), np.abs(Xg - Xo).max()))
    assert np.abs(Xg - Xo).max() <= TOL


def test_eigvec_edge_cases():
    p = make_problem(50, p2=0.25, q="householder", psel=0.5, w=8, seed=12)
    S = p.S_np().copy(order="F")
    # nothing selected: no columns
    r = sn.eigenvectors(_dev(S), None, np.zeros(50, np.int32))
    assert r["rc"] == 0 and r["ncols"] == 0
    # n = 1
    r = sn.eigenvectors(torch.full((1, 1), 3.0, dtype=torch.float64, device="cuda"), None, np.ones(1, np.int32))
    assert r["rc"] == 0 and r["ncols"] == 1 and r["X"].item() == 1.0
    # not quasi-triangular
    Sb = S.copy(order="F"); Sb[4, 1] = 1.0
    assert sn.eigenvectors(_dev(Sb), None, np.ones(50, np.int32))["rc"] == -2
    # bitwise repeatable
    sel = np.ones(50, np.int32)
    r1, X1 = _run(S, p.Q_np(), sel)
    r2, X2 = _run(S, p.Q_np(), sel)
    assert np.array_equal(X1, X2)


def test_eigvec_config3_size_sampled():
    """BASELINE config 3 (n = 40 000, Q random orthogonal, selection Bernoulli(0.35)): the GPU
    computes every selected vector, back-transformed; the oracle computes a sample of them
    (the lowest and highest blocks and a random draw -- columns are independent), compared
    elementwise; plus the residual ||A x - lambda x|| of the sampled vectors in FP64 on the
    device, A = Q S Q^T applied as Q (S (Q^T x))."""
    p = make_config(3, seed=1, device="cuda")
    n = p.n
    sel = p.select.astype(np.int32)
    r = sn.eigenvectors(p.S, p.Q, sel)
    torch.cuda.synchronize()
    assert r["rc"] == 0
    st = r["stats"]
    print("config3 eigvec: cols=%d ms_device=%.1f (backsub %.1f, backtransform %.1f) TF/s=%.2f rescales=%d" % (
        r["ncols"], st["ms_device"], st["ms_backsubstitution"], st["ms_backtransform"],
        (st["flops_update"] + st["flops_backtransform"]) / st["ms_device"] / 1e9, st["rescales"]))
    S0 = p.S.cpu().numpy().T                      # column-major view: S0[i, j] = S[i, j]
    bm = np.zeros(n, np.int8)
    sub = np.diag(S0, -1) != 0
    i = 0
    while i < n - 1:
        if sub[i]:
            bm[i], bm[i + 1] = 1, 2
            i += 2
        else:
            i += 1
    blocks = [(q, sz) for q, sz in blocks_of(bm) if sel[q] or (sz == 2 and sel[q + 1])]
    cols = np.cumsum([0] + [sz for _, sz in blocks])
    rng = np.random.default_rng(5)
    pick = sorted(set([0, len(blocks) - 1] + list(rng.choice(len(blocks), 4, replace=False))))
    sub_sel = np.zeros(n, np.int32)
    for t in pick:
        q, sz = blocks[t]
        sub_sel[q:q + sz] = 1
    Q0 = np.asfortranarray(p.Q.cpu().numpy().T)
    rc, Xo, _ = oracle.eigvec(np.asfortranarray(S0), Q0, sub_sel)
    assert rc == 0
    Xg = r["X"].cpu().numpy().T
    worst = 0.0
    c_or = 0
    for t in pick:
        q, sz = blocks[t]
        worst = max(worst, np.abs(Xg[:, cols[t]:cols[t] + sz] - Xo[:, c_or:c_or + sz]).max())
        c_or += sz
    print("config3 eigvec sampled %d vectors: max|dX| = %.3g" % (len(pick), worst))
    assert worst <= TOL
