"""Pins of the eigenvector oracle (-m "not gpu").

or_eigvec restates Eq. (5) -- back substitution for (S - lambda I) y = 0 -- with
overflow protection and the back-transform Eq. (6), readings E1-E6
(sn_oracle.c).  Pinned to things other than itself:
  * LAPACK xTREVC3 (the library routine computing exactly these vectors: selected Schur-basis
    vectors, HOWMNY='S', and back-transformed ones, 'B') through scipy's OpenBLAS;
  * closed forms (SPEC eigvec examples): diagonal S gives unit vectors; [[1, 10], [0, 2]] with
    lambda = 2 gives (10, 1) up to normalisation; a standard 2x2 block [a b; c a];
  * the defining residual ||(S - lambda I) y|| <= c n eps ||S|| ||y||, and numpy's eig on
    small inputs (the same eigenvector up to a complex factor);
  * overflow: superdiagonal entries 1e300 (SPEC) -- finite output, power-of-two scalings
    recorded, agreement with LAPACK, and the residual evaluated in exact rational arithmetic;
  * scaling invariance: S -> 2^k S leaves the normalised vectors bitwise unchanged.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from tests import lapack_ext as LX
from tests.helpers import EPS, blocks_of, bmap_from_S
from workloads import make_problem

needs_lapack = pytest.mark.skipif(not LX.available(), reason="scipy's OpenBLAS LAPACK symbols not found")


def _complex_cols(X, S, sel):
    """Columns of X as complex eigenvectors with their eigenvalues (E1 column order)."""
    out = []
    c = 0
    for r, sz in blocks_of(bmap_from_S(S)):
        if not (sel[r] or (sz == 2 and sel[r + 1])):
            continue
        if sz == 1:
            out.append((X[:, c] + 0j, S[r, r] + 0j))
        else:
            w = np.sqrt(abs(S[r, r + 1])) * np.sqrt(abs(S[r + 1, r]))
            out.append((X[:, c] + 1j * X[:, c + 1], S[r, r] + 1j * w))
        c += sz
    assert c == X.shape[1]
    return out


@needs_lapack
@pytest.mark.parametrize("n,p2,seed,frac", [(12, 0.25, 1, 1.0), (60, 0.5, 2, 0.4), (200, 0.25, 3, 1.0),
                                            (301, 0.25, 4, 0.3), (500, 0.0, 5, 0.5), (400, 1e9, 6, 0.5)])
def test_eigvec_matches_dtrevc3(n, p2, seed, frac):
    p = make_problem(n, p2=p2, q="householder", psel=0.5, w=16, seed=seed)
    S = p.S_np().copy(order="F")
    Q = p.Q_np().copy(order="F")
    sel = (np.random.default_rng(seed).random(n) < frac).astype(np.int32)
    rc, X, e = oracle.eigvec(S, None, sel)
    VR, m, info = LX.dtrevc3(S, sel)
    assert rc == 0 and info == 0 and X.shape == VR.shape
    d = np.abs(X - VR).max()
    # both normalise to max(|re| + |im|) = 1; agreement to rounding x the vectors' condition
    assert d <= 1e-11, d
    # back-transformed: all vectors, HOWMNY='B'
    rc, Xb, _ = oracle.eigvec(S, Q, np.ones(n, np.int32))
    VB, m, info = LX.dtrevc3(S, Q=Q)
    assert rc == 0 and info == 0
    assert np.abs(Xb - VB).max() <= 1e-11


def test_eigvec_closed_forms():
    S = np.asfortranarray(np.diag([1.0, 2.0, 3.0]))
    rc, X, e = oracle.eigvec(S, None, np.ones(3, np.int32))
    assert rc == 0 and np.array_equal(X, np.eye(3))
    S = np.asfortranarray([[1.0, 10.0], [0.0, 2.0]])
    rc, X, e = oracle.eigvec(S, None, np.array([0, 1], np.int32))
    # (S - 2I) y = 0: y = (10, 1) -> normalised (1, 0.1)
    assert rc == 0 and X.shape == (2, 1)
    assert X[0, 0] == 1.0 and abs(X[1, 0] - 0.1) <= EPS
    # a standard 2x2 block [a b; c a], |b| >= |c|: y = (1, i w / b) (E2)
    a, b, c = 0.5, 2.0, -0.5
    S = np.asfortranarray([[a, b], [c, a]])
    rc, X, e = oracle.eigvec(S, None, np.ones(2, np.int32))
    w = np.sqrt(abs(b * c))
    np.testing.assert_allclose(X, [[1.0, 0.0], [0.0, w / b]], atol=2 * EPS)
    # [a c; b a]: the upper entry c is the smaller one, so y = (-w / b, i) (b the lower entry)
    rc, X, e = oracle.eigvec(np.asfortranarray([[a, c], [b, a]]), None, np.ones(2, np.int32))
    np.testing.assert_allclose(X[:, 0] + 1j * X[:, 1], np.array([-w / b, 1j]) / max(w / abs(b), 1.0), atol=4 * EPS)


@pytest.mark.parametrize("n,seed", [(8, 1), (30, 2), (150, 3)])
def test_eigvec_residual_and_numpy_eig(n, seed):
    p = make_problem(n, p2=0.25, q="identity", psel=0.5, w=8, seed=seed)
    S = p.S_np().copy(order="F")
    sel = np.ones(n, np.int32)
    rc, X, e = oracle.eigvec(S, None, sel)
    assert rc == 0
    nS = np.linalg.norm(S)
    lam_np, V_np = np.linalg.eig(S)
    for y, lam in _complex_cols(X, S, sel):
        r = S @ y - lam * y
        assert np.linalg.norm(r) <= 10 * n * EPS * nS * np.linalg.norm(y)
        # numpy: the same eigenvector up to a complex factor
        j = np.argmin(np.abs(lam_np - lam))
        v = V_np[:, j]
        cosang = abs(np.vdot(v, y)) / (np.linalg.norm(v) * np.linalg.norm(y))
        assert cosang >= 1 - 1e-10


@needs_lapack
def test_eigvec_overflow_protection():
    """SPEC eigvec example: superdiagonal entries 1e300 (n = 8).  The unprotected solve
    overflows; the protected one returns finite vectors, records power-of-two scalings, agrees
    with LAPACK xTREVC3, and its residual, evaluated exactly in rational arithmetic, is at the
    rounding level of the scaled problem."""
    n = 8
    rng = np.random.default_rng(0)
    S = np.asfortranarray(np.triu(np.full((n, n), 1e300), 1) + np.diag(rng.uniform(-1, 1, n)))
    sel = np.ones(n, np.int32)
    rc, X, e = oracle.eigvec(S, None, sel)
    assert rc == 0 and np.isfinite(X).all() and e.max() > 0 and e[0] == 0
    VR, m, info = LX.dtrevc3(S, sel)
    assert np.abs(X - VR).max() <= 1e-14
    for c in range(n):
        y = X[:, c]
        lam = Fraction(S[c, c])
        res = 0.0
        for i in range(n):
            acc = Fraction(0)
            for j in range(n):
                acc += (Fraction(S[i, j]) - (lam if i == j else 0)) * Fraction(y[j])
            res = max(res, abs(float(acc)))
        assert res <= 100 * n * EPS * np.abs(S).max() * np.abs(y).max()


def test_eigvec_scaling_invariance_and_identity_Q():
    p = make_problem(120, p2=0.25, q="householder", psel=0.5, w=8, seed=9)
    S = p.S_np().copy(order="F")
    sel = (np.random.default_rng(9).random(120) < 0.5).astype(np.int32)
    rc, X, e = oracle.eigvec(S, None, sel)
    rc2, X2, e2 = oracle.eigvec(np.asfortranarray(S * 2.0 ** 40), None, sel)
    assert np.array_equal(X, X2)                        # powers of two: bitwise
    rc3, X3, e3 = oracle.eigvec(S, np.eye(120, order="F"), sel)
    np.testing.assert_allclose(X3, X, atol=4 * EPS)     # Q = I back-transform
    # a non-quasi-triangular S is rejected
    Sb = S.copy(order="F"); Sb[5, 2] = 1.0
    assert oracle.eigvec(Sb, None, sel)[0] == -2
