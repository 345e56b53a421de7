"""Pins of the bulge-chasing oracle (-m "not gpu").

or_qr_sweep restates one sweep of the small-bulge multishift QR algorithm (PAPER.md P:113-118:
bulges chased down the diagonal by overlapping 3 x 3 Householder reflectors), readings B1-B5
(sn_oracle.c).  Pinned to:
  * the implicit Q theorem: the sweep equals the explicit QR step H' = U^T H U with
    p(H) = U R, p(z) = prod (z - s_i) (Golub & Van Loan Thm 7.4.2 / Alg 7.5.1), up to the
    signs of U's columns (small numbers of shifts: the explicit product is ill-conditioned);
  * LAPACK xLAQR5 (the library routine doing one such sweep) on the same H and shifts,
    up to the signs of the basis vectors;
  * exact shifts deflate: an eigenvalue pair of H as shifts makes H'[n-2, n-3] ~ 0;
  * invariants: H' upper Hessenberg with exact zeros below the subdiagonal, Q' orthogonal,
    A = Q' H' Q'^T, eigenvalues preserved; n < 3 and no shifts are bitwise no-ops.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from tests import lapack_ext as LX
from tests.helpers import EPS

needs_lapack = pytest.mark.skipif(not LX.available(), reason="scipy's OpenBLAS LAPACK symbols not found")


def hessenberg_problem(n, rng):
    A = rng.standard_normal((n, n))
    H, Q = sla.hessenberg(A, calc_q=True)
    H = np.triu(H, -1)
    return np.asfortranarray(H), np.asfortranarray(Q)


def make_shifts(k, rng):
    """k shift pairs: conjugate pairs or two real shifts (reading B1)."""
    sr, si = [], []
    for _ in range(k):
        if rng.random() < 0.5:
            a, b = rng.uniform(-2, 2), rng.uniform(0.1, 2)
            sr += [a, a]
            si += [b, -b]
        else:
            sr += list(rng.uniform(-2, 2, 2))
            si += [0.0, 0.0]
    return np.array(sr), np.array(si)


def _signs(U, V):
    return np.where(np.einsum("ij,ij->j", U, V) < 0, -1.0, 1.0)


@pytest.mark.parametrize("n,k,seed", [(3, 1, 1), (6, 1, 2), (10, 2, 3), (16, 2, 4), (20, 3, 5)])
def test_sweep_is_the_explicit_qr_step(n, k, seed):
    rng = np.random.default_rng(seed)
    H, _ = hessenberg_problem(n, rng)
    sr, si = make_shifts(k, rng)
    rc, H1, Q1 = oracle.qr_sweep(H, np.eye(n, order="F"), sr, si)
    assert rc == 0
    M = np.eye(n)
    for j in range(0, 2 * k, 2):
        sigma, pi = sr[j] + sr[j + 1], sr[j] * sr[j + 1] - si[j] * si[j + 1]
        M = (H @ H - sigma * H + pi * np.eye(n)) @ M
    U, _ = np.linalg.qr(M)
    d = _signs(U, Q1)
    He = U.T @ H @ U
    assert np.abs(Q1 - U * d).max() <= 1e-11
    assert np.abs(H1 - d[:, None] * He * d[None, :]).max() <= 1e-11 * np.linalg.norm(H)


@needs_lapack
@pytest.mark.parametrize("n,k,seed", [(8, 1, 11), (30, 3, 12), (64, 8, 13), (150, 12, 14), (301, 20, 15)])
def test_sweep_matches_dlaqr5(n, k, seed):
    rng = np.random.default_rng(seed)
    H, Q = hessenberg_problem(n, rng)
    sr, si = make_shifts(k, rng)
    rc, H1, Q1 = oracle.qr_sweep(H, Q, sr, si)
    Hl, Ql = LX.dlaqr5(H, Q, sr.copy(), si.copy())
    d = _signs(Q.T @ Ql, Q.T @ Q1)            # signs of the basis vectors of U
    dH = np.abs(H1 - d[:, None] * Hl * d[None, :]).max() / np.linalg.norm(H)
    dQ = np.abs(Q1 - Ql * d[None, :]).max()
    assert dH <= 1e-12 and dQ <= 1e-12, (dH, dQ)


@pytest.mark.parametrize("n,seed", [(8, 21), (12, 22)])
def test_exact_shifts_deflate(n, seed):
    rng = np.random.default_rng(seed)
    H, _ = hessenberg_problem(n, rng)
    ev = np.linalg.eigvals(H)
    c = ev[np.argmax(np.abs(ev.imag))]
    assert abs(c.imag) > 0
    rc, H1, _ = oracle.qr_sweep(H, None, [c.real, c.real], [abs(c.imag), -abs(c.imag)])
    assert abs(H1[n - 2, n - 3]) <= 1e-10 * np.linalg.norm(H)
    # the deflated 2x2 block carries the shift pair
    e2 = np.sort_complex(np.linalg.eigvals(H1[n - 2:, n - 2:]))
    assert np.abs(e2 - np.sort_complex([c, np.conj(c)])).max() <= 1e-8 * np.abs(c)


@pytest.mark.parametrize("n,k,seed", [(50, 4, 31), (200, 10, 32)])
def test_sweep_invariants(n, k, seed):
    rng = np.random.default_rng(seed)
    H, Q = hessenberg_problem(n, rng)
    A = Q @ H @ Q.T
    sr, si = make_shifts(k, rng)
    rc, H1, Q1 = oracle.qr_sweep(H, Q, sr, si)
    assert rc == 0
    assert np.count_nonzero(np.tril(H1, -2)) == 0
    assert np.linalg.norm(Q1.T @ Q1 - np.eye(n)) <= 100 * n * EPS
    assert np.linalg.norm(A - Q1 @ H1 @ Q1.T) / np.linalg.norm(A) <= 100 * n * EPS
    e0 = np.sort_complex(np.linalg.eigvals(H))
    e1 = np.sort_complex(np.linalg.eigvals(H1))
    assert np.abs(e0 - e1).max() <= 1e-8 * np.abs(e0).max()
    # a row sample of Q gives those rows (B5)
    rows = np.array([0, 7, n - 1])
    rc, H2, Q2 = oracle.qr_sweep(H, np.asfortranarray(Q[rows]), sr, si)
    assert np.array_equal(H2, H1) and np.array_equal(Q2, Q1[rows])


def test_sweep_trivial_and_arguments():
    rng = np.random.default_rng(5)
    H, Q = hessenberg_problem(2, rng)
    rc, H1, Q1 = oracle.qr_sweep(H, Q, [1.0, 2.0], [0.0, 0.0])
    assert rc == 0 and np.array_equal(H1, H) and np.array_equal(Q1, Q)
    H, Q = hessenberg_problem(9, rng)
    rc, H1, Q1 = oracle.qr_sweep(H, Q, [], [])
    assert rc == 0 and np.array_equal(H1, H)
    assert oracle.qr_sweep(H, Q, [1.0], [0.0])[0] == -7                 # odd number of shifts
    assert oracle.qr_sweep(H, Q, [1.0, 2.0], [1.0, -1.0])[0] == -9       # not a conjugate pair
