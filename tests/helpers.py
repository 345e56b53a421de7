"""Invariant checks shared by the oracle pins and the GPU parity tests.

These compute properties that the mathematics fixes for ANY correct
reordering (BASELINE.json north_star invariants):
residual, orthogonality, quasi-triangular structure, stable block order and
eigenvalue preservation.  They use numpy only (no oracle, no product code).
"""
from __future__ import annotations

import numpy as np

EPS = np.finfo(np.float64).eps  # 2^-52 (c4 #14)


def blocks_of(bmap):
    """List of (row, size) from a block map (0 = 1x1, 1/2 = rows of a 2x2)."""
    out, i, n = [], 0, len(bmap)
    while i < n:
        if bmap[i] == 1:
            out.append((i, 2)); i += 2
        else:
            out.append((i, 1)); i += 1
    return out


def bmap_from_S(S):
    n = S.shape[0]
    bm = np.zeros(n, np.int8)
    i = 0
    while i < n:
        if i + 1 < n and S[i + 1, i] != 0.0:
            bm[i], bm[i + 1] = 1, 2; i += 2
        else:
            i += 1
    return bm


def block_eigs(S, r, sz):
    if sz == 1:
        return np.array([S[r, r] + 0j])
    return np.sort_complex(np.linalg.eigvals(S[r:r + 2, r:r + 2]))


def check_quasi_triangular(S, bmap):
    """Strict lower part exactly 0 except 2x2 subdiagonals; 2x2 blocks standardised."""
    n = S.shape[0]
    low = np.tril(S, -1).copy()
    for r, sz in blocks_of(bmap):
        if sz == 2:
            assert low[r + 1, r] != 0.0
            low[r + 1, r] = 0.0
            a, b, c, d = S[r, r], S[r, r + 1], S[r + 1, r], S[r + 1, r + 1]
            assert a == d, "2x2 block at %d not standardised (diagonals %r %r)" % (r, a, d)
            assert b * c < 0, "2x2 block at %d has real eigenvalues" % r
    assert np.count_nonzero(low) == 0, "nonzero below the quasi-triangular structure"


def stable_partition(sizes, flags):
    sizes, flags = np.asarray(sizes), np.asarray(flags, bool)
    order = np.concatenate([np.nonzero(flags)[0], np.nonzero(~flags)[0]])
    return order


def check_reordering(S0, Q0, sel0, S1, Q1, sel1, m, bmap1, tol_res=None, A_norm=None):
    """Full invariant set of the north star for a completed reordering.

    S0, Q0: inputs (column-major numpy, Q0 may be None = identity);
    sel0: per-row input mask; S1, Q1, sel1, m, bmap1: outputs."""
    n = S0.shape[0]
    tol = tol_res if tol_res is not None else 100 * n * EPS
    bm0 = bmap_from_S(S0)
    b0 = blocks_of(bm0)
    flags = np.array([bool(sel0[r] or (sz == 2 and sel0[r + 1])) for r, sz in b0])
    sizes = np.array([sz for _, sz in b0])
    assert m == int(sizes[flags].sum())
    # block map of the output = stable partition of the input blocks (bit exact)
    order = stable_partition(sizes, flags)
    exp_bmap = np.concatenate([[0] if sizes[t] == 1 else [1, 2] for t in order]).astype(np.int8) if n else np.zeros(0, np.int8)
    np.testing.assert_array_equal(bmap1, exp_bmap)
    np.testing.assert_array_equal(bmap_from_S(S1), exp_bmap)
    exp_sel = np.zeros(n, np.int32); exp_sel[:m] = 1
    np.testing.assert_array_equal(np.asarray(sel1, np.int32), exp_sel)
    check_quasi_triangular(S1, exp_bmap)
    # eigenvalues along the stable permutation: 1x1 bitwise, 2x2 within 1e-10 relative (c4 #13)
    b1 = blocks_of(exp_bmap)
    for (r1, sz1), t in zip(b1, order):
        r0, sz0 = b0[t]
        assert sz0 == sz1
        if sz1 == 1:
            assert S1[r1, r1] == S0[r0, r0]
        else:
            e0, e1 = block_eigs(S0, r0, 2), block_eigs(S1, r1, 2)
            assert np.max(np.abs(e0 - e1)) <= 1e-10 * max(1.0, np.max(np.abs(e0)))
    # orthogonality and residual
    Q0m = np.eye(n) if Q0 is None else Q0
    if Q1 is not None:
        orth = np.linalg.norm(Q1.T @ Q1 - np.eye(n))
        assert orth <= tol, "orthogonality %g > %g" % (orth, tol)
        A = Q0m @ S0 @ Q0m.T
        res = np.linalg.norm(A - Q1 @ S1 @ Q1.T) / max(np.linalg.norm(A), 1e-300)
        assert res <= tol, "residual %g > %g" % (res, tol)
    return order
