"""LAPACK routines scipy does not wrap (xTREVC3, xLAQR5, xLAHQR), called through ctypes from
the OpenBLAS build that ships with scipy (symbols prefixed ``scipy_``).  Test infrastructure
only: these are the library routines the oracle is pinned against (SURVEY §8c-5 "library
routines solving the same problem")."""
from __future__ import annotations

import ctypes as C
import glob
import os

import numpy as np
import scipy

_lib = None


def _load():
    global _lib
    if _lib is None:
        d = os.path.join(os.path.dirname(os.path.dirname(scipy.__file__)), "scipy.libs")
        cands = sorted(glob.glob(os.path.join(d, "libscipy_openblas*.so")))
        if not cands:
            raise OSError("scipy's OpenBLAS not found in %s" % d)
        _lib = C.CDLL(cands[0])
    return _lib


def available() -> bool:
    try:
        L = _load()
        return hasattr(L, "scipy_dtrevc3_") and hasattr(L, "scipy_dlaqr5_")
    except OSError:
        return False


def _i(v):
    return C.byref(C.c_int(int(v)))


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def dtrevc3(T, select=None, Q=None):
    """Right eigenvectors of the quasi-triangular T: HOWMNY='S' (selected, Schur basis) if
    Q is None, else 'B' (all, back-transformed by Q).  Returns (VR, m, info)."""
    L = _load()
    T = np.asfortranarray(T, dtype=np.float64).copy(order="F")
    n = T.shape[0]
    if Q is None:
        howmny = b"S"
        sel = np.ascontiguousarray(np.asarray(select) != 0, dtype=np.int32)
        mm = n
        VR = np.zeros((n, mm), order="F")
    else:
        howmny = b"B"
        sel = np.zeros(max(n, 1), np.int32)
        mm = n
        VR = np.asfortranarray(Q, dtype=np.float64).copy(order="F")
    VL = np.zeros((1, 1), order="F")
    m = C.c_int(0)
    info = C.c_int(0)
    lwork = n + 2 * n * 128 + 16
    work = np.zeros(lwork)
    L.scipy_dtrevc3_(C.c_char_p(b"R"), C.c_char_p(howmny), _p(sel), _i(n), _p(T), _i(n), _p(VL), _i(1), _p(VR),
                     _i(n), _i(mm), C.byref(m), _p(work), _i(lwork), C.byref(info), C.c_size_t(1), C.c_size_t(1))
    return VR[:, :m.value].copy(order="F"), m.value, info.value


def dlaqr5(H, Z, sr, si, ktop=0, kbot=None, kacc22=0, wantt=True):
    """One small-bulge multishift QR sweep (LAPACK xLAQR5) on H (0-based ktop..kbot inclusive)
    with the shifts sr + i si; Z accumulates the transformations (rows 0..n-1).  Returns
    (H', Z')."""
    L = _load()
    H = np.asfortranarray(H, dtype=np.float64).copy(order="F")
    Z = np.asfortranarray(Z, dtype=np.float64).copy(order="F")
    n = H.shape[0]
    kbot = n - 1 if kbot is None else kbot
    sr = np.ascontiguousarray(sr, np.float64).copy()
    si = np.ascontiguousarray(si, np.float64).copy()
    ns = len(sr)
    nbmps = ns // 2
    V = np.zeros((3, max(nbmps, 1)), order="F")
    U = np.zeros((max(3 * ns - 3, 1), max(3 * ns - 3, 1)), order="F")
    nwv = max(n, 1)
    WV = np.zeros((nwv, max(3 * ns - 3, 1)), order="F")
    WH = np.zeros((max(3 * ns - 3, 1), max(n, 1)), order="F")
    L.scipy_dlaqr5_(C.byref(C.c_int(1 if wantt else 0)), C.byref(C.c_int(1)), _i(kacc22), _i(n), _i(ktop + 1),
                    _i(kbot + 1), _i(ns), _p(sr), _p(si), _p(H), _i(n), _i(1), _i(n), _p(Z), _i(n), _p(V), _i(3),
                    _p(U), _i(U.shape[0]), _i(nwv), _p(WV), _i(nwv), _i(WH.shape[1]), _p(WH), _i(WH.shape[0]))
    return H, Z
