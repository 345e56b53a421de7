"""Seeded synthetic real Schur forms, orthogonal Q and selections (BASELINE.json configs).

The paper gives no reordering workload (SURVEY §6, P:313 describes only the
Schur-reduction inputs); BASELINE.json's generators stand in, read as in
SURVEY §8c-4 #16-20:

* S is upper quasi-triangular.  A fraction p2 of the *blocks* are 2x2:
  n2 = round(p2*n/(1+p2)) 2x2 blocks and n - 2*n2 1x1 blocks, in a seeded
  Fisher-Yates order.  1x1 eigenvalues ~ U[-10, 10].  2x2 blocks are
  standardised: equal diagonals a ~ U[-10, 10], |b|, |c| ~ U[0.5, 3],
  sign(b) a fair coin, c = -sign(b)|c| (so b*c < 0, a complex pair).
  All other strictly-upper entries iid N(0, 1); everything below the
  subdiagonal exactly 0.
* Q is I, or the product H_1 ... H_n of n Householder reflectors
  H_i = I - 2 v v^T / (v^T v) with v iid N(0, 1) (assembled in compact-WY
  blocks with fp64 torch matmuls -- harness arithmetic, not the method's).
* The selection is Bernoulli(psel) per block (a 2x2 block as a pair), or
  "trailing half": a block is selected iff its first row >= n/2.

Randomness is counter based (SplitMix64 of (seed, stream, index)), so every
entry is a pure function of its coordinates; the same code runs on CPU or
CUDA tensors.  Matrices are returned as contiguous row-major torch tensors
holding the TRANSPOSE, i.e. their memory is the column-major matrix that the
C ABI expects (``T[j, i] == S[i, j]``).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

# ---- counter-based generator ------------------------------------------------
_M64 = 1 << 64


def _s64(c: int) -> int:
    c %= _M64
    return c - _M64 if c >= (1 << 63) else c


_GOLD = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _shr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of an int64 tensor."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def _mix(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _shr(z, 30)) * _C1
    z = (z ^ _shr(z, 27)) * _C2
    return z ^ _shr(z, 31)


def _mix_int(z: int) -> int:
    z %= _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) % _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) % _M64
    return z ^ (z >> 31)


def _base(seed: int, stream: int) -> int:
    return _s64(_mix_int(_mix_int(seed * 0x100000001B3 + 0x51ED27) + stream * 0x9E3779B97F4A7C15))


def rand_bits(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """64 random bits per int64 index (SplitMix64 finaliser of a counter)."""
    return _mix((idx + 1) * _GOLD + _base(seed, stream))


def uniform(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """U[0, 1) with 53 random bits, exactly representable in fp64."""
    return _shr(rand_bits(seed, stream, idx), 11).to(torch.float64) * (2.0 ** -53)


def normal(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """N(0, 1) by Box-Muller from two counters (2*idx, 2*idx+1)."""
    u1 = (_shr(rand_bits(seed, stream, 2 * idx), 11).to(torch.float64) + 1.0) * (2.0 ** -53)
    u2 = _shr(rand_bits(seed, stream, 2 * idx + 1), 11).to(torch.float64) * (2.0 ** -53)
    return torch.sqrt(-2.0 * torch.log(u1)) * torch.cos((2.0 * math.pi) * u2)


# streams
_ST_SHUF, _ST_EIG, _ST_A, _ST_B, _ST_C, _ST_SGN, _ST_UPPER, _ST_Q, _ST_SEL = range(1, 10)
_ST_TUP, _ST_TDIAG, _ST_Z = range(10, 13)      # pencils (make_pencil)


def _uni_np(seed, stream, idx):
    return uniform(seed, stream, torch.as_tensor(np.asarray(idx, np.int64))).numpy()


# ---- configurations (BASELINE.json configs[0..4]) -------------------------------
CONFIGS = {
    0: dict(n=256, p2=0.25, q="identity", sel="bernoulli", psel=0.5, w=32),
    1: dict(n=4096, p2=0.25, q="householder", sel="bernoulli", psel=0.35, w=128),
    2: dict(n=16384, p2=0.25, q="householder", sel="bernoulli", psel=0.35, w=256),
    3: dict(n=40000, p2=0.25, q="householder", sel="bernoulli", psel=0.35, w=256),
    4: dict(n=65536, p2=0.5, q="householder", sel="trailing_half", psel=None, w=256),
}


@dataclasses.dataclass
class Problem:
    n: int
    S: torch.Tensor            # (n, n) row-major tensor holding S^T (= column-major S)
    Q: torch.Tensor | None     # same layout, or None
    select: np.ndarray         # int32 per row (block-consistent)
    w: int
    bsizes: np.ndarray         # block sizes in diagonal order (int8)
    meta: dict

    def S_np(self) -> np.ndarray:
        """Column-major numpy view (Fortran order) of S on the host."""
        return self.S.cpu().numpy().T

    def Q_np(self):
        return None if self.Q is None else self.Q.cpu().numpy().T


def block_layout(n: int, p2: float, seed: int) -> np.ndarray:
    """Block sizes in diagonal order: round(p2*n/(1+p2)) 2x2 blocks, seeded Fisher-Yates."""
    n2 = int(round(p2 * n / (1.0 + p2)))
    n2 = min(n2, n // 2)
    sizes = np.array([2] * n2 + [1] * (n - 2 * n2), dtype=np.int8)
    B = len(sizes)
    if B > 1:
        u = _uni_np(seed, _ST_SHUF, np.arange(B))
        for t in range(B - 1, 0, -1):
            j = int(u[t] * (t + 1))
            sizes[t], sizes[j] = sizes[j], sizes[t]
    return sizes


def _diag_entries(n, sizes, seed):
    """Diagonal, superdiagonal (2x2 b) and subdiagonal (2x2 c) entries."""
    B = len(sizes)
    bidx = np.arange(B)
    eig = -10.0 + 20.0 * _uni_np(seed, _ST_EIG, bidx)
    a = -10.0 + 20.0 * _uni_np(seed, _ST_A, bidx)
    bb = 0.5 + 2.5 * _uni_np(seed, _ST_B, bidx)
    cc = 0.5 + 2.5 * _uni_np(seed, _ST_C, bidx)
    sg = np.where(_uni_np(seed, _ST_SGN, bidx) < 0.5, 1.0, -1.0)
    diag = np.zeros(n); sup = {}; sub = {}
    r = 0
    starts = np.zeros(B, np.int64)
    for t in range(B):
        starts[t] = r
        if sizes[t] == 1:
            diag[r] = eig[t]
            r += 1
        else:
            diag[r] = a[t]; diag[r + 1] = a[t]
            sup[r] = sg[t] * bb[t]
            sub[r] = -sg[t] * cc[t]
            r += 2
    return diag, sup, sub, starts


def _schur_form(n, sizes, seed, device, col_block=1024):
    diag, sup, sub, starts = _diag_entries(n, sizes, seed)
    St = torch.empty((n, n), dtype=torch.float64, device=device)  # St[j, i] = S[i, j]
    rows = torch.arange(n, device=device, dtype=torch.int64)
    for c0 in range(0, n, col_block):
        c1 = min(n, c0 + col_block)
        cols = torch.arange(c0, c1, device=device, dtype=torch.int64)
        idx = cols[:, None] * n + rows[None, :]            # index of S[i, j] = i + j*n
        val = normal(seed, _ST_UPPER, idx)
        val = torch.where(rows[None, :] < cols[:, None], val, torch.zeros((), dtype=val.dtype, device=device))
        St[c0:c1] = val
    St[rows, rows] = torch.as_tensor(diag, device=device)
    if sup:
        r = torch.as_tensor(np.array(sorted(sup)), device=device)
        St[r + 1, r] = torch.as_tensor(np.array([sup[k] for k in sorted(sup)]), device=device)   # S[r, r+1]
        St[r, r + 1] = torch.as_tensor(np.array([sub[k] for k in sorted(sub)]), device=device)   # S[r+1, r]
    return St, starts


def _householder_product_T(n, seed, device, nb=128, stream=_ST_Q):
    """Returns X = Q^T (row-major tensor), so X's memory is column-major Q,
    Q = H_0 H_1 ... H_{n-1}, H_i = I - tau_i v_i v_i^T, tau_i = 2 / v_i^T v_i."""
    X = torch.eye(n, dtype=torch.float64, device=device)
    rows = torch.arange(n, device=device, dtype=torch.int64)
    for k0 in range(0, n, nb):
        k1 = min(n, k0 + nb)
        ks = torch.arange(k0, k1, device=device, dtype=torch.int64)
        V = normal(seed, stream, ks[None, :] * n + rows[:, None])     # (n, nb), column i = v_{k0+i}
        G = (V.t() @ V).cpu().numpy()
        m = k1 - k0
        tau = 2.0 / np.diag(G)
        T = np.zeros((m, m))
        for i in range(m):
            T[i, i] = tau[i]
            if i:
                T[:i, i] = -tau[i] * (T[:i, :i] @ G[:i, i])
        Tt = torch.as_tensor(T.T.copy(), device=device)
        # Q^T <- B^T Q^T with B = I - V T V^T  (so X accumulates B_last^T ... B_0^T)
        X -= V @ (Tt @ (V.t() @ X))
    return X


def make_problem(n: int, p2: float = 0.25, q: str = "householder", sel: str = "bernoulli",
                 psel: float | None = 0.35, w: int = 128, seed: int = 1, device="cpu",
                 select_blocks=None, name: str | None = None) -> Problem:
    """Generate one problem.  q in {identity, householder, none}; sel in
    {bernoulli, trailing_half, all, none, blocks} (blocks: explicit per-block flags)."""
    device = torch.device(device)
    sizes = block_layout(n, p2, seed)
    S, starts = _schur_form(n, sizes, seed, device)
    if q == "identity":
        Q = torch.eye(n, dtype=torch.float64, device=device)
    elif q == "householder":
        Q = _householder_product_T(n, seed, device)
    elif q == "none":
        Q = None
    else:
        raise ValueError(q)
    B = len(sizes)
    if sel == "bernoulli":
        flags = _uni_np(seed, _ST_SEL, np.arange(B)) < psel
    elif sel == "trailing_half":
        flags = starts >= n // 2
    elif sel == "all":
        flags = np.ones(B, bool)
    elif sel == "none":
        flags = np.zeros(B, bool)
    elif sel == "blocks":
        flags = np.asarray(select_blocks, bool)
    else:
        raise ValueError(sel)
    select = np.repeat(flags.astype(np.int32), sizes.astype(np.int64))
    meta = dict(name=name, n=n, p2=p2, q=q, sel=sel, psel=psel, w=w, seed=seed, blocks=B,
                blocks_2x2=int((sizes == 2).sum()), m=int(select.sum()))
    return Problem(n=n, S=S, Q=Q, select=select, w=w, bsizes=sizes, meta=meta)


def make_config(cfg: int, seed: int = 1, device="cpu") -> Problem:
    c = CONFIGS[cfg]
    return make_problem(c["n"], c["p2"], c["q"], c["sel"], c["psel"], c["w"], seed=seed, device=device,
                        name="config%d" % cfg)


# ---- pencils (generalized reordering) ------------------------------

@dataclasses.dataclass
class Pencil:
    n: int
    S: torch.Tensor            # (n, n) row-major tensor holding S^T (= column-major S)
    T: torch.Tensor            # same layout, upper triangular
    Q: torch.Tensor | None
    Z: torch.Tensor | None
    select: np.ndarray
    w: int
    bsizes: np.ndarray
    meta: dict

    def np(self, name):
        x = getattr(self, name)
        return None if x is None else x.cpu().numpy().T


def make_pencil(n: int, p2: float = 0.25, q: str = "householder", sel: str = "bernoulli",
                psel: float | None = 0.35, w: int = 128, seed: int = 1, device="cpu") -> Pencil:
    """A generalized real Schur form (S, T) with orthogonal Q, Z (input recipe).

    The paper has no generalized workload; the recipe extends the standard one: S exactly as
    make_problem; T upper triangular with iid N(0, 1) strictly upper entries, diagonal
    U[0.5, 2], and at the first row r of every 2x2 block of S: T[r, r+1] = 0 and T[r+1, r+1] =
    T[r, r] (the 2x2 diagonal block of T is a positive multiple of I, so the block pencil keeps
    the complex pair of S's standardised block); Q and Z independent Householder products (or
    I / None)."""
    base = make_problem(n, p2, q, sel, psel, w, seed, device)
    device = torch.device(device)
    sizes = base.bsizes
    Tt = torch.empty((n, n), dtype=torch.float64, device=device)   # Tt[j, i] = T[i, j]
    rows = torch.arange(n, device=device, dtype=torch.int64)
    for c0 in range(0, n, 1024):
        c1 = min(n, c0 + 1024)
        cols = torch.arange(c0, c1, device=device, dtype=torch.int64)
        val = normal(seed, _ST_TUP, cols[:, None] * n + rows[None, :])
        Tt[c0:c1] = torch.where(rows[None, :] < cols[:, None], val, torch.zeros((), dtype=val.dtype, device=device))
    Tt[rows, rows] = 0.5 + 1.5 * uniform(seed, _ST_TDIAG, rows)
    starts = np.concatenate([[0], np.cumsum(sizes.astype(np.int64))[:-1]])
    r2 = starts[sizes == 2]
    if len(r2):
        r = torch.as_tensor(r2, device=device)
        Tt[r + 1, r] = 0.0                                          # T[r, r+1] = 0
        Tt[r + 1, r + 1] = Tt[r, r]                                 # T[r+1, r+1] = T[r, r]
    if q == "identity":
        Z = torch.eye(n, dtype=torch.float64, device=device)
    elif q == "householder":
        Z = _householder_product_T(n, seed, device, stream=_ST_Z)
    else:
        Z = None
    meta = dict(base.meta, kind="pencil")
    return Pencil(n=n, S=base.S, T=Tt, Q=base.Q, Z=Z, select=base.select, w=w, bsizes=sizes, meta=meta)


# ---- Hessenberg inputs for the bulge-chasing sweep --------------------
_ST_HESS = 13


@dataclasses.dataclass
class Hessenberg:
    n: int
    H: torch.Tensor            # (n, n) row-major tensor holding H^T (= column-major H)
    Q: torch.Tensor | None     # same layout, or None
    sr: np.ndarray             # shifts, real parts (pairs: B1)
    si: np.ndarray             # imaginary parts
    meta: dict

    def H_np(self) -> np.ndarray:
        return self.H.cpu().numpy().T

    def Q_np(self):
        return None if self.Q is None else self.Q.cpu().numpy().T


def shift_pairs(eigs) -> tuple[np.ndarray, np.ndarray]:
    """Order eigenvalue estimates as shift pairs (reading B1): each complex conjugate pair
    together (positive imaginary part first), the real ones paired in sorted order."""
    eigs = np.asarray(eigs)
    cplx = sorted([e for e in eigs if e.imag > 0], key=lambda e: (e.real, e.imag))
    real = sorted([e.real for e in eigs if e.imag == 0])
    sr, si = [], []
    for e in cplx:
        sr += [e.real, e.real]
        si += [e.imag, -e.imag]
    if len(real) % 2:
        real = real[:-1]
    sr += real
    si += [0.0] * len(real)
    return np.array(sr, np.float64), np.array(si, np.float64)


def make_hessenberg(n: int, ns: int, q: str = "householder", seed: int = 1, device="cpu",
                    shifts: str = "random") -> Hessenberg:
    """A random upper Hessenberg matrix (entries on and above the subdiagonal iid N(0, 1),
    exact zeros below: a stand-in for the Hessenberg form of the paper's random test matrices,
    P:313), Q = I or the Householder product of make_problem, and ns shifts:
      * "random": ns/2 complex conjugate pairs, real part U[-2, 2], imaginary part U[0.1, 2]
        (seeded; the sweep's result is then a well-conditioned function of its input, so it
        is compared elementwise);
      * "trailing": the eigenvalues of the trailing ns x ns block (the xLAQR0 fall-back shift
        strategy, computed with numpy -- input generation, not the method).  Good shifts make
        subdiagonal entries nearly vanish, where the sweep's output is ill-conditioned (even
        LAPACK's xLAQR5 and the oracle then differ at O(1)): checked by invariants only."""
    device = torch.device(device)
    Ht = torch.empty((n, n), dtype=torch.float64, device=device)   # Ht[j, i] = H[i, j]
    rows = torch.arange(n, device=device, dtype=torch.int64)
    for c0 in range(0, n, 1024):
        c1 = min(n, c0 + 1024)
        cols = torch.arange(c0, c1, device=device, dtype=torch.int64)
        val = normal(seed, _ST_HESS, cols[:, None] * n + rows[None, :])
        Ht[c0:c1] = torch.where(rows[None, :] <= cols[:, None] + 1, val, torch.zeros((), dtype=val.dtype, device=device))
    if q == "identity":
        Q = torch.eye(n, dtype=torch.float64, device=device)
    elif q == "householder":
        Q = _householder_product_T(n, seed, device)
    elif q == "none":
        Q = None
    else:
        raise ValueError(q)
    if shifts == "random":
        npair = ns // 2
        re = -2.0 + 4.0 * _uni_np(seed, _ST_HESS + 1, np.arange(npair))
        im = 0.1 + 1.9 * _uni_np(seed, _ST_HESS + 2, np.arange(npair))
        sr = np.repeat(re, 2)
        si = np.stack([im, -im], 1).reshape(-1)
    elif shifts == "trailing":
        m = min(ns, n)
        tail = Ht[n - m:, n - m:].cpu().numpy().T
        sr, si = shift_pairs(np.linalg.eigvals(tail))
    else:
        raise ValueError(shifts)
    meta = dict(n=n, ns=len(sr), q=q, seed=seed, shifts=shifts)
    return Hessenberg(n=n, H=Ht, Q=Q, sr=np.ascontiguousarray(sr, np.float64),
                      si=np.ascontiguousarray(si, np.float64), meta=meta)
