"""CPU oracle for Schur-form eigenvalue reordering (ctypes binding of sn_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_1905_04975_b200`` (the product), and
the product never imports it.

Every function is a thin marshalling wrapper around the plain C in
``sn_oracle.c``; see the header ``sn_oracle.h`` for what each computes and the
PAPER.md / SPEC.md / SURVEY.md passages it follows.  Matrices are numpy fp64
arrays in Fortran (column-major) order.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sn_oracle.c")
_LIB = os.path.join(_HERE, "libsn_oracle.so")
_LIB_OMP = os.path.join(_HERE, "libsn_oracle_omp.so")
_lib = None


def build(force: bool = False, omp: bool = False) -> str:
    """Compile sn_oracle.c with plain gcc (no fast-math, no FMA contraction).  omp=True builds
    a second library with -fopenmp: the same code, its independent panel rows / columns on
    several host threads (the N-core CPU baseline)."""
    lib_path = _LIB_OMP if omp else _LIB
    if force or not os.path.exists(lib_path) or os.path.getmtime(lib_path) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "sn_oracle.h"))):
        tmp = lib_path + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fPIC", "-shared"]
                              + (["-fopenmp"] if omp else []) + ["-o", tmp, _SRC, "-lm"])
        os.replace(tmp, lib_path)
    return lib_path


class Stats(C.Structure):
    _fields_ = [("windows", C.c_int64), ("swaps", C.c_int64), ("swaps_by_type", C.c_int64 * 4),
                ("rejected_window", C.c_int64), ("rejected_swap", C.c_int64),
                ("rejected_row", C.c_int64), ("rejected_n1", C.c_int32), ("rejected_n2", C.c_int32),
                ("eq_flops", C.c_double)]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i64, i32, p = C.c_double, C.c_int64, C.c_int, C.c_void_p
        pd = C.POINTER(C.c_double)
        _lib.or_lartg.argtypes = [d, d, pd, pd, pd]
        _lib.or_larfg3.argtypes = [pd, pd, pd]
        _lib.or_lanv2.argtypes = [pd, pd, pd, pd, pd, pd]
        _lib.or_sylv.argtypes = [i32, i32, p, p, p, p, pd]
        _lib.or_sylv.restype = i32
        _lib.or_swap.argtypes = [i64, p, i64, i64, i32, i32, p, i64, i64]
        _lib.or_swap.restype = i32
        _lib.or_swap_last_reject.restype = i32
        _lib.or_scan.argtypes = [i64, p, i64, p]
        _lib.or_scan.restype = i32
        _lib.or_select.argtypes = [i64, p, p, p, C.POINTER(C.c_int64)]
        _lib.or_schedule.argtypes = [i64, p, p, i64, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                     p, p, p, p, p, p]
        _lib.or_schedule.restype = i32
        _lib.or_reorder.argtypes = [i32, i64, p, i64, p, i64, p, C.POINTER(C.c_int64), i64, i64, i64,
                                    p, C.POINTER(Stats)]
        _lib.or_reorder.restype = i32
        _lib.or_reorder_q.argtypes = [i32, i64, p, i64, p, i64, i64, p, C.POINTER(C.c_int64), i64, i64, i64,
                                      p, C.POINTER(Stats)]
        _lib.or_reorder_q.restype = i32
        _lib.or_gsylv.argtypes = [i32, i32, p, p, p, p, p, p, p, p]
        _lib.or_gsylv.restype = i32
        _lib.or_gswap.argtypes = [i64, p, i64, p, i64, i64, i32, i32, p, i64, i64, p, i64, i64]
        _lib.or_gswap.restype = i32
        _lib.or_gswap_last_variant.restype = i32
        _lib.or_eig_count.argtypes = [i64, p, i64, p, C.POINTER(C.c_int64)]
        _lib.or_eig_count.restype = i32
        _lib.or_eigvec.argtypes = [i64, p, i64, p, i64, p, p, i64, p]
        _lib.or_eigvec.restype = i32
        _lib.or_qr_sweep.argtypes = [i64, p, i64, p, i64, i64, i64, p, p]
        _lib.or_qr_sweep.restype = i32
        _lib.or_greorder.argtypes = [i32, i64, p, i64, p, i64, p, i64, p, i64, p, C.POINTER(C.c_int64),
                                     i64, i64, i64, p, C.POINTER(Stats)]
        _lib.or_greorder.restype = i32
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    a = np.asarray(a, dtype=np.float64)
    return np.asfortranarray(a)


def lartg(f: float, g: float):
    c, s, r = C.c_double(), C.c_double(), C.c_double()
    lib().or_lartg(f, g, C.byref(c), C.byref(s), C.byref(r))
    return c.value, s.value, r.value


def larfg3(alpha: float, x):
    a = C.c_double(alpha)
    xx = (C.c_double * 2)(*x)
    tau = C.c_double()
    lib().or_larfg3(C.byref(a), xx, C.byref(tau))
    return a.value, [xx[0], xx[1]], tau.value


def lanv2(a, b, c, d):
    v = [C.c_double(x) for x in (a, b, c, d)]
    cs, sn = C.c_double(), C.c_double()
    lib().or_lanv2(*[C.byref(x) for x in v], C.byref(cs), C.byref(sn))
    return tuple(x.value for x in v) + (cs.value, sn.value)


def sylv(T11, T22, T12):
    """Solve T11 X - X T22 = scale*T12; returns (X, scale, info)."""
    T11 = np.atleast_2d(np.asarray(T11, float)); T22 = np.atleast_2d(np.asarray(T22, float))
    T12 = np.atleast_2d(np.asarray(T12, float))
    n1, n2 = T11.shape[0], T22.shape[0]
    def pad(a):
        out = np.zeros((2, 2), order="F"); out[:a.shape[0], :a.shape[1]] = a; return out
    a, b, c = pad(T11), pad(T22), pad(T12.reshape(n1, n2))
    X = np.zeros((2, 2), order="F")
    scale = C.c_double()
    info = lib().or_sylv(n1, n2, _ptr(a), _ptr(b), _ptr(c), _ptr(X), C.byref(scale))
    return X[:n1, :n2].copy(), scale.value, info


def swap(T, j: int, n1: int, n2: int, Qm=None):
    """Swap adjacent blocks in place on copies; returns (rc, T', Qm')."""
    T = _f64(T).copy(order="F")
    Qc = None if Qm is None else _f64(Qm).copy(order="F")
    rc = lib().or_swap(T.shape[0], _ptr(T), T.shape[0], j, n1, n2, _ptr(Qc),
                       0 if Qc is None else Qc.shape[0], 0 if Qc is None else Qc.shape[0])
    return rc, T, Qc


def scan(S):
    S = _f64(S)
    n = S.shape[0]
    bmap = np.zeros(n, np.int8)
    rc = lib().or_scan(n, _ptr(S), max(n, 1), _ptr(bmap))
    return rc, bmap


def select(bmap, sel):
    bmap = np.ascontiguousarray(bmap, np.int8)
    sel = np.ascontiguousarray(sel, np.int32)
    out = np.zeros(len(bmap), np.int8)
    m = C.c_int64()
    lib().or_select(len(bmap), _ptr(bmap), _ptr(sel), _ptr(out), C.byref(m))
    return out, m.value


def schedule(bmap, selrow, w: int):
    """Window schedule: dict with j1, j2 (per window), off (len nwin+1), and swaps (j, n1, n2)."""
    bmap = np.ascontiguousarray(bmap, np.int8)
    selrow = np.ascontiguousarray(selrow, np.int8)
    n = len(bmap)
    nw, ns = C.c_int64(), C.c_int64()
    rc = lib().or_schedule(n, _ptr(bmap), _ptr(selrow), w, C.byref(nw), C.byref(ns),
                           None, None, None, None, None, None)
    if rc:
        raise ValueError("or_schedule rc=%d" % rc)
    j1 = np.zeros(nw.value, np.int64); j2 = np.zeros(nw.value, np.int64)
    off = np.zeros(nw.value + 1, np.int64)
    sj = np.zeros(ns.value, np.int64); s1 = np.zeros(ns.value, np.int8); s2 = np.zeros(ns.value, np.int8)
    lib().or_schedule(n, _ptr(bmap), _ptr(selrow), w, C.byref(nw), C.byref(ns),
                      _ptr(j1), _ptr(j2), _ptr(off), _ptr(sj), _ptr(s1), _ptr(s2))
    return {"j1": j1, "j2": j2, "off": off, "swap_j": sj, "swap_n1": s1, "swap_n2": s2}


def swap_last_reject() -> int:
    """Why the last swap() rejected: 0 accepted, 1 weak stability test, 2 2x2 split (R6)."""
    return lib().or_swap_last_reject()


def reorder(S, Q, select_rows, w: int, mode: int = 1, max_windows: int = -1,
            force_reject_at: int = -1, inplace: bool = False):
    """Reorder (Eq. (7)).  mode 1 = accumulated-naive (Fig. 1b), 0 = unblocked (Fig. 1a).

    Returns dict(rc, S, Q, select, m, bmap, stats).  S, Q are Fortran fp64 arrays
    (copied unless inplace=True and already Fortran fp64).  Q may hold a sample of nq <= n
    rows (shape (nq, n)): those rows of the full result (or_reorder_q)."""
    if inplace:
        assert S.dtype == np.float64 and S.flags.f_contiguous
        Sx = S
        Qx = Q
    else:
        Sx = _f64(S).copy(order="F")
        Qx = None if Q is None else _f64(Q).copy(order="F")
    n = Sx.shape[0]
    sel = np.ascontiguousarray(select_rows, np.int32).copy()
    m = C.c_int64()
    bmap = np.zeros(n, np.int8)
    st = Stats()
    nq = n if Qx is None else Qx.shape[0]
    assert Qx is None or Qx.shape[1] == n
    rc = lib().or_reorder_q(mode, n, _ptr(Sx), max(n, 1), _ptr(Qx), max(nq, 1), nq, _ptr(sel), C.byref(m), w,
                            max_windows, force_reject_at, _ptr(bmap), C.byref(st))
    stats = {f: getattr(st, f) for f, _ in Stats._fields_}
    stats["swaps_by_type"] = list(st.swaps_by_type)
    return {"rc": rc, "S": Sx, "Q": Qx, "select": sel, "m": m.value, "bmap": bmap, "stats": stats}


# ---- generalized reordering (sn_oracle.h) ---------------------------

def _pad2(a, r, c):
    out = np.zeros((2, 2), order="F")
    out[:r, :c] = np.asarray(a, float).reshape(r, c)
    return out


def gsylv(A11, A22, A12, B11, B22, B12):
    """Solve A11 R - L A22 = A12, B11 R - L B22 = B12; returns (R, L, perturbed)."""
    A11 = np.atleast_2d(np.asarray(A11, float)); A22 = np.atleast_2d(np.asarray(A22, float))
    n1, n2 = A11.shape[0], A22.shape[0]
    args = [_pad2(A11, n1, n1), _pad2(A22, n2, n2), _pad2(A12, n1, n2),
            _pad2(B11, n1, n1), _pad2(B22, n2, n2), _pad2(B12, n1, n2)]
    R = np.zeros((2, 2), order="F"); L = np.zeros((2, 2), order="F")
    info = lib().or_gsylv(n1, n2, *[_ptr(a) for a in args], _ptr(R), _ptr(L))
    return R[:n1, :n2].copy(), L[:n1, :n2].copy(), info


def gswap(S, T, j: int, n1: int, n2: int, Ql=None, Zr=None):
    """Swap adjacent blocks of the pencil (S, T) on copies; returns (rc, S', T', Ql', Zr')."""
    S = _f64(S).copy(order="F"); T = _f64(T).copy(order="F")
    Qc = None if Ql is None else _f64(Ql).copy(order="F")
    Zc = None if Zr is None else _f64(Zr).copy(order="F")
    n = S.shape[0]
    rc = lib().or_gswap(n, _ptr(S), n, _ptr(T), n, j, n1, n2,
                        _ptr(Qc), 0 if Qc is None else Qc.shape[0], 0 if Qc is None else Qc.shape[0],
                        _ptr(Zc), 0 if Zc is None else Zc.shape[0], 0 if Zc is None else Zc.shape[0])
    return rc, S, T, Qc, Zc


def gswap_last_variant() -> int:
    """Which branch the last gswap() took: 0 G1, 1 the Sylvester pair (U0, V0), 2 the left /
    3 the right re-triangularisation kept (G2/G3), -1 rejected."""
    return lib().or_gswap_last_variant()


def greorder(S, T, Q, Z, select_rows, w: int, mode: int = 1, max_windows: int = -1,
             force_reject_at: int = -1, threads: int = 0):
    """Generalized reordering (Eq. (7) right form).  Returns dict(rc, S, T, Q, Z, select, m,
    bmap, stats); all matrices Fortran fp64 copies.  threads > 0: the -fopenmp build of the
    same code, its independent panel rows / columns on that many host threads (bitwise the
    one-thread result, tests/test_oracle_generalized.py)."""
    Sx = _f64(S).copy(order="F"); Tx = _f64(T).copy(order="F")
    Qx = None if Q is None else _f64(Q).copy(order="F")
    Zx = None if Z is None else _f64(Z).copy(order="F")
    n = Sx.shape[0]
    sel = np.ascontiguousarray(select_rows, np.int32).copy()
    m = C.c_int64()
    bmap = np.zeros(n, np.int8)
    st = Stats()
    ld = max(n, 1)
    L = lib()
    if threads > 0:
        os.environ["OMP_NUM_THREADS"] = str(threads)
        L = C.CDLL(build(omp=True))
        L.or_greorder.argtypes = lib().or_greorder.argtypes
        L.or_greorder.restype = C.c_int
    rc = L.or_greorder(mode, n, _ptr(Sx), ld, _ptr(Tx), ld, _ptr(Qx), ld, _ptr(Zx), ld, _ptr(sel),
                           C.byref(m), w, max_windows, force_reject_at, _ptr(bmap), C.byref(st))
    stats = {f: getattr(st, f) for f, _ in Stats._fields_}
    stats["swaps_by_type"] = list(st.swaps_by_type)
    return {"rc": rc, "S": Sx, "T": Tx, "Q": Qx, "Z": Zx, "select": sel, "m": m.value, "bmap": bmap,
            "stats": stats}


# ---- eigenvectors (sn_oracle.h) ----------------------------------------

def eigvec(S, Q, select_rows):
    """Right eigenvectors of the selected blocks of the quasi-triangular S (Eq. (5)),
    back-transformed by Q (Eq. (6)) if given, normalised as LAPACK xTREVC.  Returns
    (rc, X (n x ncols, Fortran), scale_exp (per column))."""
    Sx = _f64(S)
    Sx = Sx if Sx.flags.f_contiguous else Sx.copy(order="F")
    n = Sx.shape[0]
    sel = np.ascontiguousarray(select_rows, np.int32)
    nc = C.c_int64()
    rc = lib().or_eig_count(n, _ptr(Sx), max(n, 1), _ptr(sel), C.byref(nc))
    if rc:
        return rc, None, None
    Qx = None if Q is None else (_f64(Q) if _f64(Q).flags.f_contiguous else _f64(Q).copy(order="F"))
    X = np.zeros((n, nc.value), order="F")
    e = np.zeros(max(nc.value, 1), np.int32)
    rc = lib().or_eigvec(n, _ptr(Sx), max(n, 1), _ptr(Qx), max(n, 1), _ptr(sel), _ptr(X), max(n, 1), _ptr(e))
    return rc, X, e[:nc.value]


# ---- bulge-chasing sweep (sn_oracle.h) ----------------------------------

def qr_sweep(H, Q, sr, si, inplace: bool = False):
    """One multishift QR sweep (readings B1-B5) on the Hessenberg H with the shifts sr + i si;
    Q (n x n, or a row sample nq x n) accumulates.  Returns (rc, H', Q')."""
    if inplace:
        Hx, Qx = H, Q
    else:
        Hx = _f64(H).copy(order="F")
        Qx = None if Q is None else _f64(Q).copy(order="F")
    n = Hx.shape[0]
    nq = n if Qx is None else Qx.shape[0]
    sr = np.ascontiguousarray(sr, np.float64)
    si = np.ascontiguousarray(si, np.float64)
    rc = lib().or_qr_sweep(n, _ptr(Hx), max(n, 1), _ptr(Qx), max(nq, 1), nq, len(sr), _ptr(sr), _ptr(si))
    return rc, Hx, Qx


def reorder_threads(S, Q, select_rows, w: int, threads: int, max_windows: int = -1, inplace: bool = False):
    """or_reorder mode 1 from the -fopenmp build on `threads` host threads (the N-core CPU
    baseline row; the same code and summation order per row / column as reorder())."""
    os.environ["OMP_NUM_THREADS"] = str(threads)
    L = C.CDLL(build(omp=True))
    L.or_reorder_q.argtypes = lib().or_reorder_q.argtypes
    L.or_reorder_q.restype = C.c_int
    Sx = S if inplace else _f64(S).copy(order="F")
    Qx = Q if (inplace or Q is None) else _f64(Q).copy(order="F")
    n = Sx.shape[0]
    sel = np.ascontiguousarray(select_rows, np.int32).copy()
    m = C.c_int64()
    bmap = np.zeros(n, np.int8)
    st = Stats()
    nq = n if Qx is None else Qx.shape[0]     # Q may hold a sample of rows, as in reorder()
    assert Qx is None or Qx.shape[1] == n
    rc = L.or_reorder_q(1, n, _ptr(Sx), max(n, 1), _ptr(Qx), max(nq, 1), nq, _ptr(sel), C.byref(m), w,
                        max_windows, -1, _ptr(bmap), C.byref(st))
    stats = {f: getattr(st, f) for f, _ in Stats._fields_}
    return {"rc": rc, "S": Sx, "Q": Qx, "select": sel, "m": m.value, "bmap": bmap, "stats": stats}
