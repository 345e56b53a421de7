"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test fixes the oracle to what the paper and the mathematics determine:
closed forms, textbook/library routines solving the same problem (LAPACK
dtrexc / dtrsen via scipy, an independent Schur decomposition), brute force
over all selections on tiny inputs, invariants, and special cases.  A dropped
term, a wrong sign or index, or a transposed operand in the oracle fails at
least one of them.  Citations: P:n = PAPER.md line, S:n = SPEC.md line.
"""
import itertools
import os

import numpy as np
import pytest
import scipy.linalg as sla
from scipy.linalg import lapack

import oracle
from tests.helpers import EPS, bmap_from_S, blocks_of, check_reordering
from workloads import make_config, make_problem

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---- Givens --------------------------------------------------------
@pytest.mark.parametrize("f,g", [(3.0, 4.0), (-3.0, 4.0), (3.0, -4.0), (1e-300, 1e-300), (1e300, 3e299),
                                 (0.0, 2.0), (0.0, -2.0), (5.0, 0.0), (-5.0, 0.0), (0.0, 0.0)])
def test_lartg_definition(f, g):
    c, s, r = oracle.lartg(f, g)
    # [c s; -s c] [f; g] = [r; 0],  c >= 0, c^2 + s^2 = 1
    assert c >= 0.0
    assert abs(c * c + s * s - 1.0) <= 4 * EPS
    scale = max(abs(f), abs(g), 1e-300)
    assert abs(c * f + s * g - r) <= 4 * EPS * scale
    assert abs(-s * f + c * g) <= 4 * EPS * scale
    if g == 0.0:
        assert (c, s, r) == (1.0, 0.0, f)
    elif f == 0.0:
        assert (c, s) == (0.0, np.sign(g)) and r == abs(g)
    else:
        assert np.sign(r) == np.sign(f)


def test_lartg_closed_form_3_4():
    assert oracle.lartg(3.0, 4.0) == (0.6, 0.8, 5.0)      # S:210 "(3,4) -> r=5"


# ---- Householder -------------------------------------------
@pytest.mark.parametrize("alpha,x", [(1.0, (0.0, 0.0)), (0.0, (0.0, 1.0)), (2.0, (-1.0, 3.0)),
                                     (-2.0, (1.0, 0.5)), (0.0, (1.0, 0.0)), (1e-200, (1e-200, 0.0))])
def test_larfg3_reflects_onto_e1(alpha, x):
    beta, v, tau = oracle.larfg3(alpha, list(x))
    a = np.array([alpha, *x])
    if x == (0.0, 0.0):
        assert tau == 0.0 and beta == alpha
        return
    vv = np.array([1.0, *v])
    H = np.eye(3) - tau * np.outer(vv, vv)
    assert np.abs(H.T @ H - np.eye(3)).max() <= 8 * EPS
    y = H @ a
    sc = np.abs(a).max()
    nrm = sc * np.linalg.norm(a / sc)
    assert abs(y[0] - beta) <= 8 * EPS * nrm and np.abs(y[1:]).max() <= 8 * EPS * nrm
    assert abs(abs(beta) - nrm) <= 4 * EPS * nrm
    assert np.sign(beta) == -(1.0 if np.copysign(1.0, alpha) > 0 else -1.0)


# ---- standardisation ---------------------------------------------------
def _lanv2_check(a, b, c, d):
    A0 = np.array([[a, b], [c, d]])
    aa, bb, cc, dd, cs, sn = oracle.lanv2(a, b, c, d)
    R = np.array([[cs, -sn], [sn, cs]])
    A1 = np.array([[aa, bb], [cc, dd]])
    assert abs(cs * cs + sn * sn - 1) <= 4 * EPS
    assert np.abs(R @ A1 @ R.T - A0).max() <= 20 * EPS * np.abs(A0).max()
    ev = np.sort_complex(np.linalg.eigvals(A0))
    if cc == 0.0:
        assert np.abs(np.sort_complex(np.array([aa, dd], complex)) - ev).max() <= 1e-12 * max(1, np.abs(ev).max())
    else:
        assert aa == dd and bb * cc < 0
    return aa, bb, cc, dd, cs, sn


def test_lanv2_already_standard_is_identity():
    assert oracle.lanv2(1.0, 2.0, -2.0, 1.0) == (1.0, 2.0, -2.0, 1.0, 1.0, 0.0)   # S:359 "1 +- 2i"


def test_lanv2_cases():
    rng = np.random.default_rng(5)
    for _ in range(500):
        a, b, c, d = rng.standard_normal(4) * rng.choice([1e-3, 1, 1e3])
        _lanv2_check(a, b, c, d)
    _lanv2_check(1.0, 0.0, 3.0, 2.0)    # b == 0: swap rows/cols
    _lanv2_check(1.0, 3.0, 0.0, 2.0)    # already triangular
    _lanv2_check(2.0, 1.0, 1.0, 2.0)    # real, equal diagonal
    _lanv2_check(1.0, -4.0, 1.0, 3.0)   # complex, unequal diagonal


# ---- small Sylvester ---------------------------------------------
@pytest.mark.parametrize("n1,n2", [(1, 2), (2, 1), (2, 2), (1, 1)])
def test_sylv_matches_library(n1, n2):
    rng = np.random.default_rng(7 + n1 * 3 + n2)
    for _ in range(50):
        T11 = rng.standard_normal((n1, n1)) * 3
        T22 = rng.standard_normal((n2, n2)) * 3 + 5
        T12 = rng.standard_normal((n1, n2))
        X, scale, info = oracle.sylv(T11, T22, T12)
        assert info == 0 and scale == 1.0
        Xref = sla.solve_sylvester(T11, -T22, T12)          # T11 X + X (-T22) = T12
        assert np.abs(X - Xref).max() <= 1e-12 * max(1, np.abs(Xref).max())
        assert np.abs(T11 @ X - X @ T22 - T12).max() <= 1e-12 * max(1, np.abs(T12).max())


def test_sylv_singular_is_perturbed():
    X, scale, info = oracle.sylv(np.eye(2), np.eye(2), np.ones((2, 2)))
    assert info == 1 and np.all(np.isfinite(X))


# ---- single swaps vs LAPACK dtrexc -----------------------------------
def _random_T(sizes, rng, upper=1.0):
    n = sum(sizes)
    T = np.triu(rng.standard_normal((n, n))) * upper
    r = 0
    for sz in sizes:
        if sz == 1:
            T[r, r] = rng.uniform(-10, 10)
        else:
            a = rng.uniform(-10, 10); b = rng.uniform(0.5, 3) * rng.choice([-1, 1]); c = -np.sign(b) * rng.uniform(0.5, 3)
            T[r, r] = T[r + 1, r + 1] = a; T[r, r + 1] = b; T[r + 1, r] = c
        r += sz
    return np.asfortranarray(T)


@pytest.mark.parametrize("n1,n2", [(1, 1), (1, 2), (2, 1), (2, 2)])
def test_swap_matches_dtrexc(n1, n2):
    rng = np.random.default_rng(100 + 10 * n1 + n2)
    worst = 0.0
    for trial in range(200):
        pre = list(rng.choice([1, 2], size=rng.integers(0, 3)))
        post = list(rng.choice([1, 2], size=rng.integers(0, 3)))
        sizes = pre + [n1, n2] + post
        T = _random_T(sizes, rng)
        n = T.shape[0]
        Q = np.asfortranarray(np.linalg.qr(rng.standard_normal((n, n)))[0])
        j = sum(pre)
        rc, T1, Q1 = oracle.swap(T, j, n1, n2, Q)
        assert rc == 0
        Tl, Ql, info = lapack.dtrexc(T.copy(), Q.copy(), j + n1 + 1, j + 1)
        assert info == 0
        assert np.array_equal(bmap_from_S(T1), bmap_from_S(Tl))
        d = max(np.abs(T1 - Tl).max() / np.linalg.norm(T), np.abs(Q1 - Ql).max())
        worst = max(worst, d)
        # the exchanged blocks: moved block's eigenvalues now lead
        e_old = np.sort_complex(np.linalg.eigvals(T[j + n1:j + n1 + n2, j + n1:j + n1 + n2]))
        e_new = np.sort_complex(np.linalg.eigvals(T1[j:j + n2, j:j + n2]))
        assert np.abs(e_old - e_new).max() <= 1e-12 * max(1, np.abs(e_old).max())
    # median agreement is ~1e-16; the worst cases (~1e-13) are moved 2x2 blocks close to a
    # scaled rotation, where the standardising rotation of lanv2 is ill-determined and both
    # LAPACK's and our (differently ordered) arithmetic give valid, slightly different forms.
    assert worst <= 1e-12, worst


def test_swap_closed_form_1x1():
    # [1 5; 0 2]: f = 5, g = 1 -> c = 5/sqrt(26), s = 1/sqrt(26); diagonals swap bitwise,
    # t12 untouched, "[1]|[2] -> swapped diagonal (2,1)".
    T = np.asfortranarray([[1.0, 5.0, 7.0], [0.0, 2.0, 3.0], [0.0, 0.0, 4.0]])
    rc, T1, Q1 = oracle.swap(T, 0, 1, 1, np.eye(3, order="F"))
    c, s = 5 / np.sqrt(26), 1 / np.sqrt(26)
    assert rc == 0 and T1[0, 0] == 2.0 and T1[1, 1] == 1.0 and T1[0, 1] == 5.0 and T1[1, 0] == 0.0
    assert abs(T1[0, 2] - (c * 7 + s * 3)) <= 4 * EPS * 10 and abs(T1[1, 2] - (c * 3 - s * 7)) <= 4 * EPS * 10
    np.testing.assert_allclose(Q1[:2, :2], [[c, -s], [s, c]], rtol=0, atol=4 * EPS)
    # f = 0: signed permutation, exact
    T = np.asfortranarray([[1.0, 0.0], [0.0, 2.0]])
    rc, T1, Q1 = oracle.swap(T, 0, 1, 1, np.eye(2, order="F"))
    assert T1.tolist() == [[2.0, 0.0], [0.0, 1.0]] and Q1.tolist() == [[0.0, -1.0], [1.0, 0.0]]
    # g = 0 ("[0]|[0]"): equal eigenvalues; the Givens path never rejects (reading R5)
    T = np.asfortranarray([[0.0, 1.0], [0.0, 0.0]])
    rc, T1, Q1 = oracle.swap(T, 0, 1, 1, np.eye(2, order="F"))
    assert rc == 0 and T1.tolist() == T.tolist() and Q1.tolist() == np.eye(2).tolist()


def test_swap_spec_example_5_and_1pm_i():
    # S:417 "{5}|{1+-i} -> {1+-i} then {5}, each within 1e-12"
    T = np.asfortranarray([[5.0, 0.3, -0.7], [0.0, 1.0, 1.0], [0.0, -1.0, 1.0]])
    rc, T1, _ = oracle.swap(T, 0, 1, 2, np.eye(3, order="F"))
    assert rc == 0
    ev = np.sort_complex(np.linalg.eigvals(T1[:2, :2]))
    assert np.abs(ev - np.array([1 - 1j, 1 + 1j])).max() <= 1e-12
    assert T1[2, 2] == 5.0 and T1[2, 0] == 0.0 and T1[2, 1] == 0.0
    assert T1[0, 0] == T1[1, 1] and T1[0, 1] * T1[1, 0] < 0


def test_swap_golden_fixtures():
    """tests/golden/swap_cases.txt: small swaps with expected values fixed by closed forms."""
    path = os.path.join(GOLDEN, "swap_cases.txt")
    cases = [l for l in open(path) if l.strip() and not l.startswith("#")]
    assert cases
    for line in cases:
        name, n, j, n1, n2, tin, tout = line.split("|")
        n, j, n1, n2 = int(n), int(j), int(n1), int(n2)
        T = np.asfortranarray(np.array([float(x) for x in tin.split()]).reshape(n, n))
        E = np.array([float(x) for x in tout.split()]).reshape(n, n)
        rc, T1, _ = oracle.swap(T, j, n1, n2, None)
        assert rc == 0, name
        assert np.abs(T1 - E).max() <= 1e-14 * max(1, np.abs(E).max()), (name, T1, E)


# ---- whole reordering vs LAPACK dtrsen (SURVEY §8c-5 row "Whole reordering", A2) --------
@pytest.mark.parametrize("mode", [0, 1])
def test_reorder_matches_dtrsen(mode):
    rng = np.random.default_rng(11)
    worst = 0.0
    cases = 0
    for seed in range(24):
        n = int(rng.integers(8, 121))
        p2 = float(rng.choice([0.0, 0.25, 0.5]))
        w = int(rng.choice([4, 6, 16, 64]))
        psel = float(rng.choice([0.2, 0.5, 0.8]))
        p = make_problem(n, p2=p2, q="householder", sel="bernoulli", psel=psel, w=w, seed=seed + 1000)
        S, Q = p.S_np(), p.Q_np()
        r = oracle.reorder(S, Q, p.select, w=w, mode=mode)
        assert r["rc"] == 0
        ts, qs, wr, wi, m, s, sep, info = lapack.dtrsen(p.select, S.copy(), Q.copy(), job="N")
        assert info == 0 and m == r["m"]
        np.testing.assert_array_equal(r["bmap"], bmap_from_S(ts))
        d = max(np.abs(r["S"] - ts).max() / np.linalg.norm(S), np.abs(r["Q"] - qs).max())
        worst = max(worst, d)
        check_reordering(S, Q, p.select, r["S"], r["Q"], r["select"], r["m"], r["bmap"])
        cases += 1
    assert worst <= 1e-12, worst


def test_modes_agree_config0_and_n1000():
    for prob in (make_config(0, seed=1), make_problem(1000, q="householder", psel=0.35, w=64, seed=3)):
        S, Q = prob.S_np(), prob.Q_np()
        a = oracle.reorder(S, Q, prob.select, w=prob.w, mode=0)
        b = oracle.reorder(S, Q, prob.select, w=prob.w, mode=1)
        np.testing.assert_array_equal(a["bmap"], b["bmap"])
        nS = np.linalg.norm(S)
        assert np.abs(a["S"] - b["S"]).max() <= 1e-12 * nS
        assert np.abs(a["Q"] - b["Q"]).max() <= 1e-11
        assert a["stats"]["swaps"] == b["stats"]["swaps"]
        check_reordering(S, Q, prob.select, b["S"], b["Q"], b["select"], b["m"], b["bmap"])


# ---- brute force on tiny inputs (BJ north_star) ------------------------------------
def test_bruteforce_all_selections_tiny():
    """All 2^B selections for n <= 12: the leading invariant subspace equals the one of an
    independent Schur decomposition of A = Q S Q^T sorted by scipy (projector equality),
    and the leading eigenvalues are exactly the selected ones."""
    for seed, n, p2 in [(1, 8, 0.25), (2, 10, 0.5), (3, 12, 0.0), (4, 9, 0.5)]:
        p = make_problem(n, p2=p2, q="householder", sel="none", w=4, seed=seed)
        S, Q = p.S_np(), p.Q_np()
        A = Q @ S @ Q.T
        blocks = blocks_of(bmap_from_S(S))
        eigs = [np.linalg.eigvals(S[r:r + sz, r:r + sz]) for r, sz in blocks]
        for mask in itertools.product([0, 1], repeat=len(blocks)):
            sel = np.repeat(np.array(mask, np.int32), [sz for _, sz in blocks])
            for w in (4, 6):
                r = oracle.reorder(S, Q, sel, w=w, mode=1)
                assert r["rc"] == 0
                check_reordering(S, Q, sel, r["S"], r["Q"], r["select"], r["m"], r["bmap"])
                m = r["m"]
                if m == 0 or m == n:
                    continue
                chosen = np.concatenate([eigs[t] for t in range(len(blocks)) if mask[t]])
                got = np.sort_complex(np.linalg.eigvals(r["S"][:m, :m]))
                assert np.abs(np.sort_complex(chosen) - got).max() <= 1e-10 * max(1, np.abs(chosen).max())

                def pick(re, im, chosen=chosen):
                    z = re + 1j * im
                    return np.min(np.abs(chosen - z)) < 1e-6
                T2, U, sdim = sla.schur(A, output="real", sort=pick)
                assert sdim == m
                P1 = U[:, :m] @ U[:, :m].T
                P2 = r["Q"][:, :m] @ r["Q"][:, :m].T
                assert np.abs(P1 - P2).max() <= 1e-10


# ---- special cases -----------------------------------------------------------------------
def test_spec_diag123_select3():
    # S:407 "s = diag(1,2,3), select {3} -> 3 in position (0,0); multiset preserved"
    S = np.asfortranarray(np.diag([1.0, 2.0, 3.0]))
    r = oracle.reorder(S, np.eye(3, order="F"), [0, 0, 1], w=4)
    assert r["rc"] == 0 and r["m"] == 1
    assert np.diag(r["S"]).tolist() == [3.0, 1.0, 2.0]
    assert np.count_nonzero(r["S"] - np.diag(np.diag(r["S"]))) == 0
    assert sorted(np.abs(r["Q"]).ravel().tolist()) == [0.0] * 6 + [1.0] * 3


@pytest.mark.parametrize("mode", [0, 1])
def test_block_diagonal_is_exact_signed_block_permutation(mode):
    """S with zero coupling: every transform is a signed (block) permutation,
    so the result is exact: S-blocks and Q-columns move as signed permutations."""
    for seed, n, p2 in [(1, 50, 0.0), (2, 60, 0.25), (3, 120, 0.5)]:
        p = make_problem(n, p2=p2, q="householder", sel="bernoulli", psel=0.4, w=16, seed=seed)
        S0 = p.S_np().copy(order="F")
        bm = bmap_from_S(S0)
        mask = np.zeros_like(S0, bool)
        for rr, sz in blocks_of(bm):
            mask[rr:rr + sz, rr:rr + sz] = True
        S0[~mask] = 0.0
        Q0 = p.Q_np()
        r = oracle.reorder(S0, Q0, p.select, w=16, mode=mode)
        order = check_reordering(S0, Q0, p.select, r["S"], r["Q"], r["select"], r["m"], r["bmap"])
        b0, b1 = blocks_of(bm), blocks_of(r["bmap"])
        off = np.ones_like(S0, bool)
        for (r1, sz), t in zip(b1, order):
            r0 = b0[t][0]
            off[r1:r1 + sz, r1:r1 + sz] = False
            found = False
            for perm in itertools.permutations(range(sz)):
                for signs in itertools.product([1.0, -1.0], repeat=sz):
                    P = np.zeros((sz, sz))
                    for a, b_ in enumerate(perm):
                        P[b_, a] = signs[a]
                    if (np.array_equal(r["S"][r1:r1 + sz, r1:r1 + sz], P.T @ S0[r0:r0 + sz, r0:r0 + sz] @ P)
                            and (mode == 0 and p2 > 0 or np.array_equal(r["Q"][:, r1:r1 + sz], Q0[:, r0:r0 + sz] @ P))):
                        found = True
            assert found, (seed, r1, r0)
        assert np.count_nonzero(r["S"][off]) == 0


def test_trivial_selections_are_bitwise_noops():
    p = make_problem(64, q="householder", sel="all", w=8, seed=5)
    S, Q = p.S_np(), p.Q_np()
    for sel in (p.select, np.zeros_like(p.select)):
        r = oracle.reorder(S, Q, sel, w=8)
        assert r["rc"] == 0 and r["stats"]["windows"] == 0
        assert np.array_equal(r["S"], S) and np.array_equal(r["Q"], Q)
    # already leading
    sel = np.zeros_like(p.select); sel[:10] = 1
    if bmap_from_S(S)[9] == 1:
        sel[10] = 1
    r = oracle.reorder(S, Q, sel, w=8)
    assert r["stats"]["windows"] == 0 and np.array_equal(r["S"], S)
    # n = 0, 1
    r = oracle.reorder(np.zeros((1, 1), order="F") + 3.0, np.eye(1, order="F"), [1], w=4)
    assert r["rc"] == 0 and r["m"] == 1


def test_idempotent():
    p = make_problem(200, q="householder", psel=0.35, w=32, seed=9)
    r = oracle.reorder(p.S_np(), p.Q_np(), p.select, w=32)
    r2 = oracle.reorder(r["S"], r["Q"], r["select"], w=32)
    assert r2["stats"]["windows"] == 0
    assert np.array_equal(r2["S"], r["S"]) and np.array_equal(r2["Q"], r["Q"])


def test_argument_errors():
    S = np.asfortranarray(np.diag([1.0, 2.0]))
    S2 = S.copy(order="F"); S2[1, 0] = 1.0; S3 = np.asfortranarray(np.zeros((3, 3))); S3[2, 0] = 1.0
    assert oracle.reorder(S3, None, [0, 0, 1], w=4)["rc"] == -3
    assert oracle.reorder(S, None, [0, 1], w=2)["rc"] == -9
    S4 = np.asfortranarray(np.triu(np.ones((4, 4)))); S4[1, 0] = 1.0; S4[2, 1] = 1.0
    assert oracle.reorder(S4, None, [0, 0, 0, 1], w=4)["rc"] == -3


# ---- schedule -----------------------------------------------
def test_schedule_single_mover_covering():
    # S:425 "single selected 1x1 block at the bottom of a 10x10 -> ceil(distance/stride) windows"
    for w in (4, 5, 6, 10, 16):
        bmap = np.zeros(10, np.int8)
        sel = np.zeros(10, np.int8); sel[9] = 1
        sch = oracle.schedule(bmap, sel, w)
        stride = w - 1
        assert len(sch["j1"]) == -(-9 // stride)
        assert len(sch["swap_j"]) == 9
        assert np.all(sch["j2"] - sch["j1"] <= w)


def test_schedule_properties_config0():
    p = make_config(0, seed=1)
    bm = bmap_from_S(p.S_np())
    sel, m = oracle.select(bm, p.select)
    sch = oracle.schedule(bm, sel, p.w)
    k = sch["j2"] - sch["j1"]
    assert np.all(k <= p.w) and np.all(k >= 2)
    for t in range(len(k)):
        a, b = sch["off"][t], sch["off"][t + 1]
        assert b > a
        sj, s1, s2 = sch["swap_j"][a:b], sch["swap_n1"][a:b], sch["swap_n2"][a:b]
        assert np.all(sj >= sch["j1"][t]) and np.all(sj + s1 + s2 <= sch["j2"][t])
    # every (selected, unselected-above) pair is swapped exactly once
    blocks = blocks_of(bm)
    flags = [bool(sel[r]) for r, _ in blocks]
    pairs = 0
    uns = 0
    for f in flags:
        if f:
            pairs += uns
        else:
            uns += 1
    assert len(sch["swap_j"]) == pairs


# ---- failure path (SURVEY §8b +1) ----------------------------------------------
@pytest.mark.parametrize("mode", [0, 1])
def test_forced_rejection_leaves_consistent_state(mode):
    p = make_problem(150, p2=0.25, q="householder", psel=0.4, w=16, seed=21)
    S, Q = p.S_np(), p.Q_np()
    full = oracle.reorder(S, Q, p.select, w=16, mode=mode)
    at = full["stats"]["swaps"] // 2
    r = oracle.reorder(S, Q, p.select, w=16, mode=mode, force_reject_at=at)
    assert r["rc"] == 1 and r["stats"]["rejected_swap"] == at and r["stats"]["swaps"] == at
    n = S.shape[0]
    A = Q @ S @ Q.T
    assert np.linalg.norm(A - r["Q"] @ r["S"] @ r["Q"].T) / np.linalg.norm(A) <= 100 * n * EPS
    assert np.linalg.norm(r["Q"].T @ r["Q"] - np.eye(n)) <= 100 * n * EPS
    np.testing.assert_array_equal(r["bmap"], bmap_from_S(r["S"]))
    assert int(r["select"].sum()) == r["m"]
    # the selected 1x1 eigenvalues are still present in the reported selected rows
    assert r["select"][r["stats"]["rejected_row"] + r["stats"]["rejected_n1"]] == 1


# ---- natural rejections: the weak test (c4 #5) and the 2x2 split (R6)
def _near_pair(rng, n1, n2):
    """Adjacent blocks with nearly equal eigenvalues (pairs lam +- i mu, mu in [1e-9, 1e-3])
    and a coupling up to 1e8: ill-conditioned Sylvester equations, where LAPACK dtrexc
    rejects (info = 1) or splits a moved 2x2 block into two real eigenvalues."""
    lam, mu, big = rng.uniform(-1, 1), 10 ** rng.uniform(-9, -3), 10 ** rng.uniform(0, 8)

    def blk2(l, m):
        b = rng.uniform(0.5, 2)
        return np.array([[l, b], [-m * m / b, l]])
    n = n1 + n2
    T = np.zeros((n, n))
    near = lambda: lam + rng.uniform(-1, 1) * mu  # noqa: E731
    if n1 == 1:
        T[0, 0] = near()
    else:
        T[:2, :2] = blk2(lam, mu)
    if n2 == 1:
        T[n1, n1] = near()
    else:
        T[n1:, n1:] = blk2(near(), mu * rng.uniform(0.5, 2))
    T[:n1, n1:] = rng.standard_normal((n1, n2)) * big
    return np.asfortranarray(T)


@pytest.mark.parametrize("n1,n2", [(2, 1), (2, 2)])
def test_natural_rejections_match_dtrexc(n1, n2):
    """Without any forcing: where LAPACK dtrexc rejects the swap (info = 1) the oracle's weak
    test rejects it (reason 1); where dtrexc splits a moved 2x2 block, the oracle rejects by
    reading R6 (reason 2); where dtrexc swaps normally, the oracle swaps.  Rejected swaps leave
    T and Q bitwise untouched."""
    rng = np.random.default_rng(5 + 10 * n1 + n2)
    n = n1 + n2
    tab = {}
    for _ in range(1500):
        T = _near_pair(rng, n1, n2)
        Tl, _, info = lapack.dtrexc(T.copy(), np.eye(n), n1 + 1, 1)
        exp = [False] * (n - 1)
        if n2 == 2:
            exp[0] = True
        if n1 == 2:
            exp[n2] = True
        split = [bool(Tl[i + 1, i] != 0) for i in range(n - 1)] != exp
        lap = 1 if info else (2 if split else 0)
        rc, T1, Q1 = oracle.swap(T, 0, n1, n2, np.eye(n, order="F"))
        why = oracle.swap_last_reject()
        assert rc == (1 if why else 0)
        if rc:
            assert np.array_equal(T1, T) and np.array_equal(Q1, np.eye(n))
        tab[(lap, why)] = tab.get((lap, why), 0) + 1
    agree = sum(v for (a, b), v in tab.items() if a == b)
    print((n1, n2), tab)
    assert agree >= 0.99 * 1500, tab
    assert tab.get((2, 2), 0) >= 100                       # the split branch fires
    if n1 == 2 and n2 == 2:
        assert tab.get((1, 1), 0) >= 100                   # the weak test fires


def test_natural_rejection_in_reordering_matches_dtrsen():
    """A whole reordering that must pass an ill-conditioned 2x2|2x2 pair: LAPACK dtrsen
    fails (info = 1) and so does the oracle (rc = 1, both modes), leaving a valid partially
    reordered form and reporting the pair."""
    rng = np.random.default_rng(77)
    for _ in range(200):
        B = _near_pair(rng, 2, 2)
        if lapack.dtrexc(B.copy(), np.eye(4), 3, 1)[2] == 1:
            break
    n = 7
    S = np.triu(rng.standard_normal((n, n)))
    S[0, 0], S[1, 1], S[2, 2] = 4.0, -3.0, 6.5
    S[3:, 3:] = B
    S = np.asfortranarray(S)
    Q = np.asfortranarray(np.linalg.qr(rng.standard_normal((n, n)))[0])
    sel = np.zeros(n, np.int32)
    sel[5] = sel[6] = 1                                    # the lower 2x2 block must pass the upper
    *_, info = lapack.dtrsen(sel, S.copy(), Q.copy(), job="N")
    assert info == 1
    for mode in (0, 1):
        r = oracle.reorder(S, Q, sel, w=8, mode=mode)
        assert r["rc"] == 1 and r["stats"]["rejected_row"] == 3 and r["stats"]["rejected_n1"] == 2
        A = Q @ S @ Q.T
        assert np.linalg.norm(A - r["Q"] @ r["S"] @ r["Q"].T) / np.linalg.norm(A) <= 100 * n * EPS
        np.testing.assert_array_equal(r["bmap"], bmap_from_S(r["S"]))
        assert r["select"][5:7].sum() == 2 and r["m"] == 2   # the block stopped below the pair


def test_row_sampled_Q_gives_those_rows():
    """or_reorder_q: a row sample of Q yields exactly those rows of the full result (the
    rows of Q <- Q Q3 are independent), used for prefix parity at config 4."""
    p = make_problem(300, p2=0.25, q="householder", psel=0.4, w=32, seed=3)
    S0, Q0 = p.S_np().copy(order="F"), p.Q_np().copy(order="F")
    rows = np.array([0, 5, 77, 150, 299])
    for mode in (0, 1):
        a = oracle.reorder(S0, Q0, p.select, w=32, mode=mode)
        b = oracle.reorder(S0, np.asfortranarray(Q0[rows]), p.select, w=32, mode=mode)
        assert np.array_equal(a["S"], b["S"]) and np.array_equal(a["Q"][rows], b["Q"])


def test_threaded_oracle_is_bitwise_the_oracle():
    """The -fopenmp build (the N-core CPU baseline row) runs the same code: every panel row /
    column keeps its summation order, so the result is bitwise the single-thread oracle's."""
    p = make_problem(700, p2=0.25, q="householder", psel=0.35, w=64, seed=41)
    S0, Q0 = p.S_np().copy(order="F"), p.Q_np().copy(order="F")
    a = oracle.reorder(S0, Q0, p.select, w=64)
    b = oracle.reorder_threads(S0, Q0, p.select, 64, 4)
    assert a["rc"] == b["rc"] == 0
    assert np.array_equal(a["S"], b["S"]) and np.array_equal(a["Q"], b["Q"])
    np.testing.assert_array_equal(a["bmap"], b["bmap"])


def test_threaded_oracle_prefix_and_q_sample_bitwise():
    """reorder_threads with max_windows and a row sample of Q (the GPU full-size prefix tests'
    arguments) is bitwise reorder() with the same arguments."""
    p = make_problem(600, p2=0.5, q="householder", psel=0.35, w=64, seed=43)
    S0, Q0 = p.S_np().copy(order="F"), p.Q_np().copy(order="F")
    rows = np.array([1, 44, 300, 599])
    for Qa in (Q0, np.asfortranarray(Q0[rows])):
        a = oracle.reorder(S0, Qa, p.select, w=64, max_windows=7)
        b = oracle.reorder_threads(S0, Qa, p.select, 64, 3, max_windows=7)
        assert a["rc"] == b["rc"] == 0 and a["stats"]["windows"] == 7
        assert np.array_equal(a["S"], b["S"]) and np.array_equal(a["Q"], b["Q"])
