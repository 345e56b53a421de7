"""Pins of the generalized-reordering oracle against things other than itself.

PAPER.md Eq. (7), right form: (S, T) = Q3 (Ŝ, T̂) Z3^T; Table 1 lists
generalized reordering beside the standard case.  The oracle (oracle/sn_oracle.c, or_gsylv /
or_gswap / or_greorder, readings G1-G6) is pinned to:
  * LAPACK dtgsyl (generalized Sylvester), dtgexc (one swap) and dtgsen (whole reordering) via
    scipy -- an independent implementation of the same textbook method: every entry agrees in
    absolute value (signs of basis vectors are a convention), the deflating subspaces agree as
    projectors;
  * the Kronecker form of the Sylvester pair solved by numpy;
  * invariants: Q (Ŝ, T̂) Z^T = (S, T), orthogonality, exact structure, eigenvalues moved along
    the stable partition;
  * special cases: T = I reduces to the standard reordering (pinned in test_oracle_pins.py);
    block-diagonal pencils are exact signed block permutations.
A dropped term, a wrong sign or index, or a transposed operand in any step fails one of them.
"""
import numpy as np
import pytest
import scipy.linalg as sla
from scipy.linalg import lapack

import oracle
from tests.helpers import EPS, bmap_from_S, blocks_of, stable_partition
from workloads import make_pencil, make_problem


def _rand_pencil(sizes, rng, upper=1.0):
    """Generalized real Schur form: S quasi-triangular with standardised 2x2 blocks, T upper
    triangular with a positive multiple of I on each 2x2 block (so the pair stays complex)."""
    n = sum(sizes)
    S = np.triu(rng.standard_normal((n, n))) * upper
    T = np.triu(rng.standard_normal((n, n))) * upper
    r = 0
    for sz in sizes:
        if sz == 1:
            S[r, r] = rng.uniform(-10, 10)
            T[r, r] = rng.uniform(0.5, 2)
        else:
            a = rng.uniform(-10, 10); b = rng.uniform(0.5, 3) * rng.choice([-1, 1]); c = -np.sign(b) * rng.uniform(0.5, 3)
            S[r, r] = S[r + 1, r + 1] = a; S[r, r + 1] = b; S[r + 1, r] = c
            T[r, r] = T[r + 1, r + 1] = rng.uniform(0.5, 2); T[r, r + 1] = 0.0
        r += sz
    return np.asfortranarray(S), np.asfortranarray(T)


def _orth(n, rng):
    return np.asfortranarray(np.linalg.qr(rng.standard_normal((n, n)))[0])


def _proj(X):
    q, _ = np.linalg.qr(X)
    return q @ q.T


def _geig(S, T):
    return np.array(sorted(sla.eigvals(S, T), key=lambda z: (round(z.imag, 8), z.real)))


def check_gstructure(S, T):
    """Generalized real Schur form: S quasi-triangular, T upper triangular (exact zeros), every
    2x2 block of T diagonal with t11 >= t22 > 0 and its pencil a complex pair, every 1x1 block
    of T nonnegative (G4)."""
    bm = bmap_from_S(S)
    low = np.tril(S, -1).copy()
    for r, sz in blocks_of(bm):
        if sz == 1:
            assert T[r, r] >= 0.0
        if sz == 2:
            low[r + 1, r] = 0.0
            assert T[r, r + 1] == 0.0 and T[r, r] >= T[r + 1, r + 1] > 0.0
            e = sla.eigvals(S[r:r + 2, r:r + 2], T[r:r + 2, r:r + 2])
            assert abs(e[0].imag) > 0
    assert np.count_nonzero(low) == 0
    assert np.count_nonzero(np.tril(T, -1)) == 0
    return bm


def check_greordering(S0, T0, Q0, Z0, sel0, r, tol=None):
    """North-star invariants for a completed generalized reordering (result dict r)."""
    n = S0.shape[0]
    tol = tol if tol is not None else 100 * n * EPS
    b0 = blocks_of(bmap_from_S(S0))
    flags = np.array([bool(sel0[q] or (sz == 2 and sel0[q + 1])) for q, sz in b0])
    sizes = np.array([sz for _, sz in b0])
    assert r["m"] == int(sizes[flags].sum())
    order = stable_partition(sizes, flags)
    exp_bmap = np.concatenate([[0] if sizes[t] == 1 else [1, 2] for t in order]).astype(np.int8)
    np.testing.assert_array_equal(r["bmap"], exp_bmap)
    np.testing.assert_array_equal(check_gstructure(r["S"], r["T"]), exp_bmap)
    for (r1, sz1), t in zip(blocks_of(exp_bmap), order):
        r0, sz0 = b0[t]
        e0 = _geig(S0[r0:r0 + sz0, r0:r0 + sz0], T0[r0:r0 + sz0, r0:r0 + sz0])
        e1 = _geig(r["S"][r1:r1 + sz1, r1:r1 + sz1], r["T"][r1:r1 + sz1, r1:r1 + sz1])
        assert np.abs(e0 - e1).max() <= 1e-10 * max(1.0, np.abs(e0).max())
    Q1, Z1 = r["Q"], r["Z"]
    assert np.linalg.norm(Q1.T @ Q1 - np.eye(n)) <= tol
    assert np.linalg.norm(Z1.T @ Z1 - np.eye(n)) <= tol
    for X0, X1 in ((S0, r["S"]), (T0, r["T"])):
        A = Q0 @ X0 @ Z0.T
        assert np.linalg.norm(A - Q1 @ X1 @ Z1.T) / np.linalg.norm(A) <= tol


# ---- generalized Sylvester pair (G2) ---------------------------------------------------
@pytest.mark.parametrize("n1,n2", [(1, 1), (1, 2), (2, 1), (2, 2)])
def test_gsylv_matches_dtgsyl_and_kronecker(n1, n2):
    rng = np.random.default_rng(7 + 10 * n1 + n2)
    for _ in range(50):
        S, T = _rand_pencil([n1, n2], rng)
        A11, A22, A12 = S[:n1, :n1], S[n1:, n1:], S[:n1, n1:]
        B11, B22, B12 = T[:n1, :n1], T[n1:, n1:], T[:n1, n1:]
        R, L, pert = oracle.gsylv(A11, A22, A12, B11, B22, B12)
        assert pert == 0
        # LAPACK: A R - L B = scale C, D R - L E = scale F
        Rl, Ll, scale, dif, info = lapack.dtgsyl(A11, A22, A12, B11, B22, B12)
        assert info == 0
        np.testing.assert_allclose(R, Rl / scale, rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(L, Ll / scale, rtol=1e-11, atol=1e-12)
        # Kronecker form, column-major vec
        I1, I2 = np.eye(n1), np.eye(n2)
        K = np.block([[np.kron(I2, A11), -np.kron(A22.T, I1)], [np.kron(I2, B11), -np.kron(B22.T, I1)]])
        x = np.linalg.solve(K, np.concatenate([A12.flatten("F"), B12.flatten("F")]))
        N = n1 * n2
        np.testing.assert_allclose(R.flatten("F"), x[:N], rtol=1e-11, atol=1e-12)
        np.testing.assert_allclose(L.flatten("F"), x[N:], rtol=1e-11, atol=1e-12)


def test_gsylv_common_eigenvalue_is_perturbed():
    # (S11, T11) and (S22, T22) share the eigenvalue 2: the Kronecker matrix is singular
    R, L, pert = oracle.gsylv([[2.0]], [[4.0]], [[1.0]], [[1.0]], [[2.0]], [[1.0]])
    assert pert == 1 and np.all(np.isfinite(R)) and np.all(np.isfinite(L))


# ---- one swap vs LAPACK dtgexc (G1-G4) ---------------------------------------------------
@pytest.mark.parametrize("n1,n2", [(1, 1), (1, 2), (2, 1), (2, 2)])
def test_gswap_matches_dtgexc(n1, n2):
    rng = np.random.default_rng(300 + 10 * n1 + n2)
    worst_el = worst_proj = 0.0
    variants = {}
    for _ in range(300):
        pre = list(rng.choice([1, 2], size=rng.integers(0, 3)))
        post = list(rng.choice([1, 2], size=rng.integers(0, 3)))
        S, T = _rand_pencil(pre + [n1, n2] + post, rng)
        n = S.shape[0]
        Q, Z = _orth(n, rng), _orth(n, rng)
        j = sum(pre)
        rc, S1, T1, Q1, Z1 = oracle.gswap(S, T, j, n1, n2, Q, Z)
        assert rc == 0
        variants[oracle.gswap_last_variant()] = variants.get(oracle.gswap_last_variant(), 0) + 1
        # G7: with Z = I the swap's right factor sits in columns j..j+n1+n2; the largest-
        # magnitude entry of each of its columns is positive
        _, _, _, _, Zi = oracle.gswap(S, T, j, n1, n2, None, np.eye(n, order="F"))
        for c in range(j, j + n1 + n2):
            col = Zi[j:j + n1 + n2, c]
            assert col[np.argmax(np.abs(col))] > 0
        a, b, ql, zl, _, info = lapack.dtgexc(S.copy(), T.copy(), Q.copy(), Z.copy(), j + n1 + 1, j + 1)
        assert info == 0
        np.testing.assert_array_equal(bmap_from_S(S1), bmap_from_S(a))
        check_gstructure(S1, T1)
        worst_el = max(worst_el, np.abs(np.abs(S1) - np.abs(a)).max() / np.linalg.norm(S),
                       np.abs(np.abs(T1) - np.abs(b)).max() / np.linalg.norm(T))
        k = j + n2
        worst_proj = max(worst_proj, np.abs(_proj(Q1[:, :k]) - _proj(ql[:, :k])).max(),
                         np.abs(_proj(Z1[:, :k]) - _proj(zl[:, :k])).max())
        # the moved block's generalized eigenvalues now lead
        e_old = _geig(S[j + n1:j + n1 + n2, j + n1:j + n1 + n2], T[j + n1:j + n1 + n2, j + n1:j + n1 + n2])
        e_new = _geig(S1[j:j + n2, j:j + n2], T1[j:j + n2, j:j + n2])
        assert np.abs(e_old - e_new).max() <= 1e-12 * max(1, np.abs(e_old).max())
        # backward stability of the swap
        for X0, X1 in ((S, S1), (T, T1)):
            assert np.abs(Q1 @ X1 @ Z1.T - Q @ X0 @ Z.T).max() <= 20 * EPS * np.linalg.norm(X0)
        assert np.abs(Q1.T @ Q1 - np.eye(n)).max() <= 20 * EPS
        assert np.abs(Z1.T @ Z1 - np.eye(n)).max() <= 20 * EPS
    assert worst_el <= 1e-12, worst_el
    assert worst_proj <= 1e-12, worst_proj
    print((n1, n2), "variants kept:", variants)
    if (n1, n2) != (1, 1):
        # every G2 candidate -- the Sylvester pair and both re-triangularisations of xTGEX2 --
        # is kept in some of these swaps, and each matches dtgexc (the former G2b
        # branch had no pin)
        assert min(variants.get(q, 0) for q in (1, 2, 3)) >= 5, variants


def test_gswap_identity_T_is_the_standard_swap():
    # T = I: the pencil swap is the standard swap (pinned in test_oracle_pins.py) with U = V;
    # 1x1|1x1 gives the same Givens rotation, the other types the same invariant subspaces
    rng = np.random.default_rng(41)
    for n1, n2 in [(1, 1), (1, 2), (2, 1), (2, 2)]:
        for _ in range(40):
            S, _T = _rand_pencil([n1, n2, 1], rng)
            n = S.shape[0]
            I = np.asfortranarray(np.eye(n))
            rc, S1, T1, Q1, Z1 = oracle.gswap(S, I, 0, n1, n2, I, I)
            rs, S2, Q2 = oracle.swap(S, 0, n1, n2, I)
            assert rc == 0 and rs == 0
            np.testing.assert_allclose(T1, np.eye(n), atol=20 * EPS)
            np.testing.assert_allclose(Q1, Z1, atol=20 * EPS)
            assert np.abs(_proj(Q1[:, :n2]) - _proj(Q2[:, :n2])).max() <= 1e-13
            if n1 == n2 == 1:
                # the same rotation up to the basis-sign convention G7 (largest-magnitude
                # entry of each column of the right factor positive)
                d = np.ones(n)
                for c in range(2):
                    d[c] = np.sign(Q2[np.argmax(np.abs(Q2[:, c])), c])
                np.testing.assert_allclose(S1, d[:, None] * S2 * d[None, :], atol=1e-14 * np.abs(S).max())
                np.testing.assert_allclose(Q1, Q2 * d[None, :], atol=1e-15)


def test_gswap_rejects_real_pair_and_keeps_state():
    # a 1x1|2x2 pencil whose 2x2 block has a complex pair but a near-identical 1x1 eigenvalue
    # still swaps; a 2x2 block of T that is singular rejects (G4) and changes nothing
    S = np.asfortranarray([[1.0, 0.3, 0.2], [0.0, 2.0, 1.0], [0.0, -1.0, 2.0]])
    T = np.asfortranarray([[1.0, 0.5, 0.1], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    rc, S1, T1, _, _ = oracle.gswap(S, T, 0, 1, 2)
    assert rc == 0
    Ts = T.copy(order="F"); Ts[1, 1] = Ts[2, 2] = 0.0     # infinite eigenvalues: T block singular
    rc, S2, T2, _, _ = oracle.gswap(S, Ts, 0, 1, 2)
    assert rc == 1 and np.array_equal(S2, S) and np.array_equal(T2, Ts)


# ---- whole reordering vs LAPACK dtgsen (G5, G6) -----------------------------------------
@pytest.mark.parametrize("mode", [0, 1])
def test_greorder_matches_dtgsen(mode):
    rng = np.random.default_rng(12)
    worst_el = worst_proj = 0.0
    for seed in range(14):
        n = int(rng.integers(8, 101))
        p2 = float(rng.choice([0.0, 0.25, 0.5]))
        w = int(rng.choice([4, 6, 16, 64]))
        psel = float(rng.choice([0.2, 0.5, 0.8]))
        p = make_pencil(n, p2=p2, q="householder", sel="bernoulli", psel=psel, w=w, seed=seed + 2000)
        S, T, Q, Z = p.np("S"), p.np("T"), p.np("Q"), p.np("Z")
        r = oracle.greorder(S, T, Q, Z, p.select, w=w, mode=mode)
        assert r["rc"] == 0
        a, b, _, _, _, qs, zs, m, _, _, _, info = lapack.dtgsen(p.select, S.copy(), T.copy(), Q.copy(), Z.copy(), ijob=0)
        assert info == 0 and m == r["m"]
        check_greordering(S, T, Q, Z, p.select, r)
        worst_el = max(worst_el, np.abs(np.abs(r["S"]) - np.abs(a)).max() / np.linalg.norm(S),
                       np.abs(np.abs(r["T"]) - np.abs(b)).max() / np.linalg.norm(T))
        if m:
            worst_proj = max(worst_proj, np.abs(_proj(r["Q"][:, :m]) - _proj(qs[:, :m])).max(),
                             np.abs(_proj(r["Z"][:, :m]) - _proj(zs[:, :m])).max())
    assert worst_el <= 1e-12, worst_el
    assert worst_proj <= 1e-12, worst_proj


def test_greorder_identity_T_matches_standard_subspace():
    p = make_problem(200, q="householder", psel=0.35, w=32, seed=5)
    S, Q = p.S_np(), p.Q_np()
    I = np.asfortranarray(np.eye(200))
    g = oracle.greorder(S, I, Q, Q, p.select, w=32, mode=1)
    s = oracle.reorder(S, Q, p.select, w=32, mode=1)
    assert g["rc"] == 0 == s["rc"] and g["m"] == s["m"]
    np.testing.assert_array_equal(g["bmap"], s["bmap"])
    m = s["m"]
    assert np.abs(_proj(g["Q"][:, :m]) - _proj(s["Q"][:, :m])).max() <= 1e-11
    assert np.abs(_proj(g["Z"][:, :m]) - _proj(s["Q"][:, :m])).max() <= 1e-11
    np.testing.assert_allclose(g["T"], np.eye(200), atol=1e-12)


def test_greorder_modes_agree():
    p = make_pencil(300, p2=0.25, q="householder", psel=0.35, w=32, seed=9)
    S, T, Q, Z = p.np("S"), p.np("T"), p.np("Q"), p.np("Z")
    r0 = oracle.greorder(S, T, Q, Z, p.select, w=32, mode=0)
    r1 = oracle.greorder(S, T, Q, Z, p.select, w=32, mode=1)
    assert r0["rc"] == 0 == r1["rc"]
    check_greordering(S, T, Q, Z, p.select, r1)
    for key in ("S", "T"):
        assert np.abs(r0[key] - r1[key]).max() <= 1e-12 * np.linalg.norm(r0[key])
    for key in ("Q", "Z"):
        assert np.abs(r0[key] - r1[key]).max() <= 1e-12


@pytest.mark.parametrize("mode", [0, 1])
def test_greorder_block_diagonal_is_signed_block_permutation(mode):
    # no coupling: every swap is an exchange, so |Ŝ|, |T̂| are the block permutation.  The
    # exchanges are exact signed permutations in exact arithmetic; G2's re-triangularisations
    # (Householder QR of a permuted diagonal block, xTGEX2) round at the ulp level, so the
    # comparison is to a few eps instead of bitwise (the standard path stays bitwise)
    rng = np.random.default_rng(3)
    sizes = list(rng.choice([1, 2], size=40))
    S, T = _rand_pencil(sizes, rng, upper=0.0)
    n = S.shape[0]
    sel_blocks = rng.random(len(sizes)) < 0.5
    select = np.repeat(sel_blocks.astype(np.int32), sizes)
    I = np.asfortranarray(np.eye(n))
    r = oracle.greorder(S, T, I, I, select, w=8, mode=mode)
    assert r["rc"] == 0
    b0 = blocks_of(bmap_from_S(S))
    order = stable_partition([sz for _, sz in b0], sel_blocks)
    Sp = np.zeros_like(S); Tp = np.zeros_like(T)
    r1 = 0
    for t in order:
        r0, sz = b0[t]
        Sp[r1:r1 + sz, r1:r1 + sz] = S[r0:r0 + sz, r0:r0 + sz]
        Tp[r1:r1 + sz, r1:r1 + sz] = T[r0:r0 + sz, r0:r0 + sz]
        r1 += sz
    tol = 16 * EPS
    assert np.abs(r["T"] - Tp).max() <= tol * np.abs(T).max()     # t >= 0, 2x2 blocks t*I
    # S: the block permutation up to basis signs.  A 2x2 block of T equal to t*I leaves its S
    # block determined only up to an orthogonal similarity (G4's SVD is degenerate there, and
    # the ulp-level rounding picks the rotation): its generalized eigenvalues and Frobenius
    # norm are compared instead
    d = np.abs(r["S"]) - np.abs(Sp)
    blk_cols = np.zeros(n, int)
    src_rows = {}
    r1 = 0
    for t in order:
        r0, sz = b0[t]
        src_rows[r1] = (r0, sz)
        r1 += sz
    for r1, sz in blocks_of(bmap_from_S(Sp)):
        if sz == 2:
            e0 = np.sort_complex(sla.eigvals(Sp[r1:r1 + 2, r1:r1 + 2], Tp[r1:r1 + 2, r1:r1 + 2]))
            e1 = np.sort_complex(sla.eigvals(r["S"][r1:r1 + 2, r1:r1 + 2], r["T"][r1:r1 + 2, r1:r1 + 2]))
            assert np.abs(e0 - e1).max() <= 1e-13 * np.abs(e0).max()
            assert abs(np.linalg.norm(r["S"][r1:r1 + 2, r1:r1 + 2]) - np.linalg.norm(Sp[r1:r1 + 2, r1:r1 + 2])) \
                <= tol * np.abs(S).max()
            d[r1:r1 + 2, r1:r1 + 2] = 0.0
    assert np.abs(d).max() <= tol * np.abs(S).max()
    # Q, Z: nonzero only on the block permutation's pattern (column block <- its source rows)
    for key in ("Q", "Z"):
        mask = np.zeros((n, n), bool)
        for r1, (r0, sz) in src_rows.items():
            mask[r0:r0 + sz, r1:r1 + sz] = True
        assert np.abs(r[key][~mask]).max() <= tol
        np.testing.assert_allclose(r[key].T @ r[key], np.eye(n), atol=tol)


@pytest.mark.parametrize("mode", [0, 1])
def test_greorder_forced_rejection_leaves_consistent_state(mode):
    p = make_pencil(120, p2=0.25, q="householder", psel=0.4, w=16, seed=4)
    S, T, Q, Z = p.np("S"), p.np("T"), p.np("Q"), p.np("Z")
    r = oracle.greorder(S, T, Q, Z, p.select, w=16, mode=mode, force_reject_at=500)
    assert r["rc"] == 1 and r["stats"]["rejected_swap"] == 500
    n = S.shape[0]
    bm = check_gstructure(r["S"], r["T"])
    np.testing.assert_array_equal(bm, r["bmap"])
    for X0, X1 in ((S, r["S"]), (T, r["T"])):
        A = Q @ X0 @ Z.T
        assert np.linalg.norm(A - r["Q"] @ X1 @ r["Z"].T) / np.linalg.norm(A) <= 100 * n * EPS


def test_greorder_argument_errors():
    p = make_pencil(20, w=8, seed=1)
    S, T, Q, Z = p.np("S"), p.np("T"), p.np("Q"), p.np("Z")
    Tb = T.copy(order="F"); Tb[5, 2] = 1e-300
    assert oracle.greorder(S, Tb, Q, Z, p.select, w=8)["rc"] == -5
    assert oracle.greorder(S, T, Q, Z, p.select, w=3)["rc"] == -13
    r = oracle.greorder(S, T, None, None, p.select, w=8)
    assert r["rc"] == 0


def test_greorder_inwindow_order_independence():
    # reading R12 for pencils: the GPU executes each window's swaps in the product's order
    # (inner windows, movers top to bottom; sn_schedule_window_swaps, host code) -- the same
    # block pairs as the oracle's mover-by-mover order.  Applying the oracle's own swap in that
    # order must give the oracle's result to rounding, up to basis-vector signs.
    import ctypes as C
    import paper_1905_04975_b200 as sn
    p = make_pencil(160, p2=0.25, q="householder", psel=0.4, w=32, seed=21)
    S, T, Q, Z = (p.np(x).copy(order="F") for x in ("S", "T", "Q", "Z"))
    ref = oracle.greorder(S, T, Q, Z, p.select, w=32, mode=0)
    assert ref["rc"] == 0
    rc, bmap = oracle.scan(S)
    selrow, _ = oracle.select(bmap, p.select)
    nwin = len(sn.schedule(bmap, selrow, 32)["j1"])
    L, n = oracle.lib(), S.shape[0]
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)   # noqa: E731
    for t in range(nwin):
        sj, s1, s2 = sn.window_swaps(bmap, selrow, 32, t)
        for j, a1, a2 in zip(sj, s1, s2):
            assert L.or_gswap(n, ptr(S), n, ptr(T), n, int(j), int(a1), int(a2), ptr(Q), n, n, ptr(Z), n, n) == 0
    dQ = np.where(np.einsum("ij,ij->j", Q, ref["Q"]) < 0, -1.0, 1.0)
    dZ = np.where(np.einsum("ij,ij->j", Z, ref["Z"]) < 0, -1.0, 1.0)
    assert np.abs(S - dQ[:, None] * ref["S"] * dZ[None, :]).max() <= 1e-11 * np.linalg.norm(S)
    assert np.abs(T - dQ[:, None] * ref["T"] * dZ[None, :]).max() <= 1e-11 * np.linalg.norm(T)
    assert np.abs(Q - ref["Q"] * dQ).max() <= 1e-11 and np.abs(Z - ref["Z"] * dZ).max() <= 1e-11


def test_greorder_threaded_is_bitwise_the_oracle():
    """The -fopenmp build of or_greorder (used by the GPU tests at the config-1/2 pencil sizes)
    runs the same code, every panel row / column keeping its summation order: bitwise the
    one-thread result, with and without a window prefix."""
    p = make_pencil(420, p2=0.25, q="householder", psel=0.4, w=64, seed=17)
    S, T, Q, Z = p.np("S"), p.np("T"), p.np("Q"), p.np("Z")
    for mw in (-1, 5):
        a = oracle.greorder(S, T, Q, Z, p.select, w=64, max_windows=mw)
        b = oracle.greorder(S, T, Q, Z, p.select, w=64, max_windows=mw, threads=3)
        assert a["rc"] == b["rc"] == 0
        for key in ("S", "T", "Q", "Z"):
            assert np.array_equal(a[key], b[key]), key
        np.testing.assert_array_equal(a["bmap"], b["bmap"])
