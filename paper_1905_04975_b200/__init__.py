"""B200-native eigenvalue reordering of a real Schur form (arXiv 1905.04975, Eq. (7)).

Thin ctypes binding of ``libsn_b200.so`` (C ABI: ``include/sn_reorder.h``).  Argument
marshalling only: every step of the reordering runs in the library's CUDA kernels.  There
is no CPU fallback -- if the shared library is missing, importing this package raises.

Matrices are passed as torch tensors whose memory is the column-major matrix, i.e. a
contiguous row-major tensor ``T`` with ``T[j, i] == S[i, j]`` (see ``workloads``), either
on ``cuda`` (fast path, in place) or on the CPU (staged through the GPU inside the call).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
LIB_PATH = os.path.join(_HERE, "libsn_b200.so")
# A/B timing tools only: load another prebuilt in-tree copy of the library (never rebuilt)
_LIB_OVERRIDE = os.environ.get("SN_LIB_PATH")
if _LIB_OVERRIDE:
    LIB_PATH = os.path.abspath(_LIB_OVERRIDE)
CSRC = os.path.join(_HERE, "csrc")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the CUDA library for sm_100a (nvcc; works without a GPU)."""
    if _LIB_OVERRIDE:
        return LIB_PATH
    srcs = sources()
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps.append(os.path.join(_ROOT, "include", "sn_reorder.h"))
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= max(map(os.path.getmtime, deps)):
        return LIB_PATH
    tmp = LIB_PATH + ".tmp%d" % os.getpid()
    cmd = ["nvcc", *NVCC_FLAGS, "-shared", "-I", os.path.join(_ROOT, "include"), "-o", tmp, *srcs]
    out = subprocess.run(cmd, capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + out.stderr[-6000:])
    if verbose:
        print(out.stderr)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class Opts(C.Structure):
    _fields_ = [("window", C.c_int64), ("inner_window", C.c_int64), ("max_windows", C.c_int64),
                ("force_reject_window", C.c_int64), ("force_reject_swap", C.c_int64),
                ("validate_lower", C.c_int32), ("serialize", C.c_int32), ("q_stream_overlap", C.c_int32),
                ("profile", C.c_int32), ("lookahead", C.c_int32), ("fuse_chain", C.c_int32),
                ("pencil_cluster", C.c_int32)]


class Stats(C.Structure):
    _fields_ = [("windows", C.c_int64), ("levels", C.c_int64), ("swaps", C.c_int64),
                ("swaps_by_type", C.c_int64 * 4), ("inner_windows", C.c_int64),
                ("rejected_window", C.c_int64), ("rejected_row", C.c_int64),
                ("rejected_n1", C.c_int32), ("rejected_n2", C.c_int32),
                ("eq_flops", C.c_double), ("ms_schedule", C.c_double), ("ms_device", C.c_double),
                ("ms_total", C.c_double), ("ms_h2d", C.c_double), ("ms_d2h", C.c_double),
                ("launches", C.c_int64 * 5), ("ms_kernel", C.c_double * 5), ("flops_kernel", C.c_double * 5),
                ("bytes_kernel", C.c_double * 5), ("flops_exec_kernel", C.c_double * 5),
                ("g3_max_ratio", C.c_double), ("fused_q_pairs", C.c_int64)]

    def to_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        for f in ("swaps_by_type", "launches", "ms_kernel", "flops_kernel", "bytes_kernel", "flops_exec_kernel"):
            d[f] = list(getattr(self, f))
        return d


SN_OK, SN_ERR_REJECTED, SN_ERR_CUDA, SN_ERR_NCCL, SN_ERR_UNSUPPORTED = 0, 1, 2, 3, 4

EXPORTS = ["sn_default_opts", "sn_strerror", "sn_reorder_schur", "sn_reorder_schur_ex",
           "sn_schedule_build", "sn_schedule_lookahead", "sn_schedule_window_swaps", "sn_version",
           "sn_dist_unique_id", "sn_dist_init", "sn_dist_finalize", "sn_dist_layout", "sn_reorder_schur_dist",
           "sn_reorder_schur_dist_local", "sn_dist_program", "sn_release_workspace", "sn_reorder_pencil_ex",
           "sn_eigenvectors", "sn_sweep_default_opts", "sn_qr_sweep", "sn_sweep_schedule"]


class SweepOpts(C.Structure):
    _fields_ = [("window", C.c_int64), ("bulges_per_chain", C.c_int64), ("q_stream_overlap", C.c_int32),
                ("lookahead", C.c_int32)]


class SweepStats(C.Structure):
    _fields_ = [("windows", C.c_int64), ("levels", C.c_int64), ("chains", C.c_int64), ("bulges", C.c_int64),
                ("launches", C.c_int64), ("eq_flops", C.c_double), ("flops_left", C.c_double),
                ("flops_right", C.c_double), ("flops_q", C.c_double), ("ms_device", C.c_double),
                ("ms_total", C.c_double)]

    def to_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class EigStats(C.Structure):
    _fields_ = [("columns", C.c_int64), ("vectors", C.c_int64), ("tiles", C.c_int64), ("rescales", C.c_int64),
                ("launches", C.c_int64), ("flops_solve", C.c_double), ("flops_update", C.c_double),
                ("flops_backtransform", C.c_double), ("ms_backsubstitution", C.c_double),
                ("ms_backtransform", C.c_double), ("ms_normalize", C.c_double), ("ms_device", C.c_double),
                ("ms_total", C.c_double)]

    def to_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}

_lib = None


def lib():
    """Load libsn_b200.so (fails loudly if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libsn_b200.so not built: run paper_1905_04975_b200.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        i64, p = C.c_int64, C.c_void_p
        L.sn_default_opts.argtypes = [C.POINTER(Opts)]
        L.sn_strerror.argtypes = [C.c_int]
        L.sn_strerror.restype = C.c_char_p
        L.sn_version.restype = C.c_char_p
        L.sn_reorder_schur.argtypes = [i64, p, i64, p, i64, p, C.POINTER(i64)]
        L.sn_reorder_schur.restype = C.c_int
        L.sn_reorder_schur_ex.argtypes = [C.POINTER(Opts), i64, p, i64, p, i64, p, C.POINTER(i64), p,
                                          C.POINTER(Stats), p]
        L.sn_reorder_schur_ex.restype = C.c_int
        L.sn_schedule_build.argtypes = [i64, p, p, i64, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64),
                                        p, p, p, p]
        L.sn_schedule_build.restype = C.c_int
        L.sn_schedule_lookahead.argtypes = [i64, p, p, i64, i64, p, p]
        L.sn_schedule_lookahead.restype = C.c_int
        L.sn_schedule_window_swaps.argtypes = [i64, p, p, i64, i64, i64, i64, p, p, p]
        L.sn_schedule_window_swaps.restype = i64
        L.sn_dist_unique_id.argtypes = [p]
        L.sn_dist_unique_id.restype = C.c_int
        L.sn_dist_init.argtypes = [C.c_int, C.c_int, p, C.c_int]
        L.sn_dist_init.restype = C.c_int
        L.sn_dist_finalize.restype = C.c_int
        L.sn_dist_layout.argtypes = [i64, i64, i64, i64, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
        L.sn_dist_layout.restype = C.c_int
        L.sn_reorder_schur_dist.argtypes = [C.POINTER(Opts), i64, i64, p, i64, p, i64, p, C.POINTER(i64), p,
                                            C.POINTER(Stats), p]
        L.sn_reorder_schur_dist.restype = C.c_int
        L.sn_reorder_schur_dist_local.argtypes = [C.POINTER(Opts), i64, i64, i64, p, i64, p, i64, p, C.POINTER(i64),
                                                  p, C.POINTER(Stats), p]
        L.sn_reorder_schur_dist_local.restype = C.c_int
        L.sn_dist_program.argtypes = [i64, p, p, i64, i64, i64, i64, i64, p]
        L.sn_dist_program.restype = i64
        L.sn_reorder_pencil_ex.argtypes = [C.POINTER(Opts), i64, p, i64, p, i64, p, i64, p, i64, p, C.POINTER(i64),
                                           p, C.POINTER(Stats), p]
        L.sn_reorder_pencil_ex.restype = C.c_int
        L.sn_eigenvectors.argtypes = [i64, p, i64, p, i64, p, p, i64, C.POINTER(i64), p, C.POINTER(EigStats), p]
        L.sn_eigenvectors.restype = C.c_int
        L.sn_sweep_default_opts.argtypes = [C.POINTER(SweepOpts)]
        L.sn_qr_sweep.argtypes = [i64, p, i64, p, i64, i64, p, p, C.POINTER(SweepOpts), C.POINTER(SweepStats), p]
        L.sn_qr_sweep.restype = C.c_int
        L.sn_sweep_schedule.argtypes = [i64, i64, i64, i64, C.POINTER(i64), C.POINTER(i64), p, p, p, p, p, p]
        L.sn_sweep_schedule.restype = C.c_int
        _lib = L
    return _lib


def default_opts(**kw) -> Opts:
    o = Opts()
    lib().sn_default_opts(C.byref(o))
    for k, v in kw.items():
        setattr(o, k, v)
    return o


def strerror(code: int) -> str:
    return lib().sn_strerror(code).decode()


def _tensor_ptr(t):
    if t is None:
        return None, 0
    import torch
    assert t.dtype == torch.float64 and t.dim() == 2 and t.shape[0] == t.shape[1] and t.is_contiguous(), \
        "expect a contiguous square fp64 tensor holding the transposed (column-major) matrix"
    return C.c_void_p(t.data_ptr()), t.shape[0]


def sn_reorder_schur(n, S, ldS, Q, ldQ, select, stream=None):
    """The BASELINE signature sn_reorder_schur(n, S, ldS, Q, ldQ, select, &m) on raw pointers.

    S, Q: integer addresses (device or host); select: np.int32 array (in/out).
    Returns (rc, m)."""
    m = C.c_int64()
    sel = np.ascontiguousarray(select, np.int32)
    rc = lib().sn_reorder_schur(n, C.c_void_p(S), ldS, None if Q is None else C.c_void_p(Q), ldQ,
                                sel.ctypes.data_as(C.c_void_p), C.byref(m))
    if isinstance(select, np.ndarray) and select.dtype == np.int32 and select.flags.c_contiguous:
        select[:] = sel
    return rc, m.value


def reorder(S, Q, select, window: int = 256, stream=None, **opts):
    """Reorder in place.  S, Q: torch fp64 tensors (column-major memory, see module doc), Q
    may be None.  select: per-row int32 mask (copied).  Returns dict(rc, m, select, bmap,
    stats)."""
    import torch
    ps, n = _tensor_ptr(S)
    pq, nq = _tensor_ptr(Q)
    if Q is not None:
        assert nq == n and Q.device == S.device
    o = default_opts(window=window, **opts)
    sel = np.ascontiguousarray(select, np.int32).copy()
    bmap = np.zeros(n, np.int8)
    m = C.c_int64()
    st = Stats()
    if stream is None and S.is_cuda:
        stream = torch.cuda.current_stream(S.device).cuda_stream
    rc = lib().sn_reorder_schur_ex(C.byref(o), n, ps, n, pq, n, sel.ctypes.data_as(C.c_void_p), C.byref(m),
                                   bmap.ctypes.data_as(C.c_void_p), C.byref(st),
                                   None if stream is None else C.c_void_p(stream))
    return {"rc": rc, "m": m.value, "select": sel, "bmap": bmap, "stats": st.to_dict()}


def eigenvectors(S, Q, select, stream=None, scale_exp=False):
    """Right eigenvectors of the selected blocks of the real Schur form S (Eq. (5)),
    back-transformed by Q (Eq. (6)) if given (sn_eigenvectors, row f4).  S, Q: CUDA fp64
    tensors holding the transposed (column-major) matrices.  Returns dict(rc, X, ncols,
    scale_exp, stats); X is a CUDA tensor of shape (ncols, n) holding X^T (column j of X is
    row j of the tensor)."""
    import torch
    ps, n = _tensor_ptr(S)
    pq, nq = _tensor_ptr(Q)
    assert Q is None or nq == n
    sel = np.ascontiguousarray(select, np.int32)
    nc = C.c_int64()
    L = lib()
    if stream is None and S.is_cuda:
        stream = torch.cuda.current_stream(S.device).cuda_stream
    sv = None if stream is None else C.c_void_p(stream)
    rc = L.sn_eigenvectors(n, ps, n, pq, n, sel.ctypes.data_as(C.c_void_p), None, n, C.byref(nc), None, None, sv)
    if rc:
        return {"rc": rc, "X": None, "ncols": 0, "scale_exp": None, "stats": None}
    X = torch.empty((max(nc.value, 1), n), dtype=torch.float64, device=S.device)
    e = np.zeros(max(nc.value, 1), np.int32)
    st = EigStats()
    rc = L.sn_eigenvectors(n, ps, n, pq, n, sel.ctypes.data_as(C.c_void_p), C.c_void_p(X.data_ptr()), n,
                           C.byref(nc), e.ctypes.data_as(C.c_void_p) if scale_exp else None, C.byref(st), sv)
    return {"rc": rc, "X": X[:nc.value], "ncols": nc.value, "scale_exp": e[:nc.value] if scale_exp else None,
            "stats": st.to_dict()}


def qr_sweep(H, Q, sr, si, stream=None, **opts):
    """One multishift QR bulge-chasing sweep in place (sn_qr_sweep, row f3).  H, Q: CUDA fp64
    tensors holding the transposed (column-major) matrices; Q may be None.  sr, si: the
    shifts.  Returns dict(rc, stats)."""
    import torch
    ph, n = _tensor_ptr(H)
    pq, nq = _tensor_ptr(Q)
    assert Q is None or nq == n
    o = SweepOpts()
    lib().sn_sweep_default_opts(C.byref(o))
    for k, v in opts.items():
        setattr(o, k, v)
    sr = np.ascontiguousarray(sr, np.float64)
    si = np.ascontiguousarray(si, np.float64)
    st = SweepStats()
    if stream is None and H.is_cuda:
        stream = torch.cuda.current_stream(H.device).cuda_stream
    rc = lib().sn_qr_sweep(n, ph, n, pq, n, len(sr), sr.ctypes.data_as(C.c_void_p), si.ctypes.data_as(C.c_void_p),
                           C.byref(o), C.byref(st), None if stream is None else C.c_void_p(stream))
    return {"rc": rc, "stats": st.to_dict()}


def sweep_schedule(n: int, nshift: int, window: int = 160, bulges_per_chain: int = 16):
    """Host-only: the windows of one sweep (w0, k, level, chain, tau0, tau1) in sequential order."""
    nw, nl = C.c_int64(), C.c_int64()
    L = lib()
    rc = L.sn_sweep_schedule(n, nshift, window, bulges_per_chain, C.byref(nw), C.byref(nl), None, None, None,
                             None, None, None)
    if rc:
        raise ValueError("sn_sweep_schedule rc=%d" % rc)
    out = {key: np.zeros(nw.value, np.int64) for key in ("w0", "k", "level", "chain", "tau0", "tau1")}
    L.sn_sweep_schedule(n, nshift, window, bulges_per_chain, C.byref(nw), C.byref(nl),
                        *[out[key].ctypes.data_as(C.c_void_p) for key in ("w0", "k", "level", "chain", "tau0", "tau1")])
    out["nlevels"] = nl.value
    return out


def reorder_pencil(S, T, Q, Z, select, window: int = 256, stream=None, **opts):
    """Generalized reordering in place (sn_reorder_pencil_ex).  S, T, Q, Z: CUDA torch fp64
    tensors (column-major memory, see module doc); Q and/or Z may be None.  Returns dict(rc, m,
    select, bmap, stats)."""
    import torch
    ps, n = _tensor_ptr(S)
    pt, nt = _tensor_ptr(T)
    pq, nq = _tensor_ptr(Q)
    pz, nz = _tensor_ptr(Z)
    assert nt == n and (Q is None or nq == n) and (Z is None or nz == n)
    o = default_opts(window=window, **opts)
    sel = np.ascontiguousarray(select, np.int32).copy()
    bmap = np.zeros(n, np.int8)
    m = C.c_int64()
    st = Stats()
    if stream is None and S.is_cuda:
        stream = torch.cuda.current_stream(S.device).cuda_stream
    rc = lib().sn_reorder_pencil_ex(C.byref(o), n, ps, n, pt, n, pq, n, pz, n, sel.ctypes.data_as(C.c_void_p),
                                    C.byref(m), bmap.ctypes.data_as(C.c_void_p), C.byref(st),
                                    None if stream is None else C.c_void_p(stream))
    return {"rc": rc, "m": m.value, "select": sel, "bmap": bmap, "stats": st.to_dict()}


def schedule(bmap, selrow, w: int):
    """Host-only: the windows the library executes (schedule order)."""
    bmap = np.ascontiguousarray(bmap, np.int8)
    selrow = np.ascontiguousarray(selrow, np.int8)
    n = len(bmap)
    nw, ns, nl = C.c_int64(), C.c_int64(), C.c_int64()
    L = lib()
    rc = L.sn_schedule_build(n, bmap.ctypes.data_as(C.c_void_p), selrow.ctypes.data_as(C.c_void_p), w,
                             C.byref(nw), C.byref(ns), C.byref(nl), None, None, None, None)
    if rc:
        raise ValueError("sn_schedule_build rc=%d" % rc)
    j1, k, lev, sw = (np.zeros(nw.value, np.int64) for _ in range(4))
    L.sn_schedule_build(n, bmap.ctypes.data_as(C.c_void_p), selrow.ctypes.data_as(C.c_void_p), w,
                        C.byref(nw), C.byref(ns), C.byref(nl), j1.ctypes.data_as(C.c_void_p),
                        k.ctypes.data_as(C.c_void_p), lev.ctypes.data_as(C.c_void_p), sw.ctypes.data_as(C.c_void_p))
    return {"j1": j1, "k": k, "level": lev, "nswap": sw, "nlevels": nl.value, "total_swaps": ns.value}


def lookahead(bmap, selrow, w: int, strip: int = 64):
    """Host-only: per window (schedule order) the critical left/right strip counts."""
    bmap = np.ascontiguousarray(bmap, np.int8)
    selrow = np.ascontiguousarray(selrow, np.int8)
    nw = len(schedule(bmap, selrow, w)["j1"])
    cl = np.zeros(nw, np.int32); cr = np.zeros(nw, np.int32)
    rc = lib().sn_schedule_lookahead(len(bmap), bmap.ctypes.data_as(C.c_void_p), selrow.ctypes.data_as(C.c_void_p),
                                     w, strip, cl.ctypes.data_as(C.c_void_p), cr.ctypes.data_as(C.c_void_p))
    if rc:
        raise ValueError("sn_schedule_lookahead rc=%d" % rc)
    return cl, cr


def window_swaps(bmap, selrow, w: int, t: int, inner_window: int = 64):
    bmap = np.ascontiguousarray(bmap, np.int8)
    selrow = np.ascontiguousarray(selrow, np.int8)
    n = len(bmap)
    cap = w * w
    sj = np.zeros(cap, np.int64); s1 = np.zeros(cap, np.int8); s2 = np.zeros(cap, np.int8)
    cnt = lib().sn_schedule_window_swaps(n, bmap.ctypes.data_as(C.c_void_p), selrow.ctypes.data_as(C.c_void_p),
                                         w, inner_window, t, cap, sj.ctypes.data_as(C.c_void_p),
                                         s1.ctypes.data_as(C.c_void_p), s2.ctypes.data_as(C.c_void_p))
    if cnt < 0:
        raise ValueError("sn_schedule_window_swaps rc=%d" % cnt)
    return sj[:cnt], s1[:cnt], s2[:cnt]


# ---- sharded (multi-GPU) reordering: include/sn_reorder.h "sharded" section ----------------

def dist_layout(n: int, P: int, col_block: int, rank: int):
    """(user_cols, q0, q1): this rank's S_loc columns and Q row range (host only)."""
    uc, q0, q1 = C.c_int64(), C.c_int64(), C.c_int64()
    rc = lib().sn_dist_layout(n, P, col_block, rank, C.byref(uc), C.byref(q0), C.byref(q1))
    if rc:
        raise ValueError("sn_dist_layout rc=%d" % rc)
    return uc.value, q0.value, q1.value


def owned_columns(n: int, P: int, col_block: int, rank: int) -> np.ndarray:
    """Global columns of rank's blocks in local (compact layout) order."""
    nb = (n + col_block - 1) // col_block
    return np.concatenate([np.arange(b * col_block, min(n, (b + 1) * col_block)) for b in range(rank, nb, P)]
                          or [np.zeros(0, np.int64)]).astype(np.int64)


def shard(S, Q, P: int, col_block: int, rank: int):
    """Rank's shards of full S, Q (torch tensors holding the column-major matrices, as in
    reorder()): S_loc (user_cols, n) and Q_loc (n, ldq) tensors whose memory is the
    column-major n x user_cols block columns and (q1-q0) x n row block (ldq = ceil(n/P)
    rounded up to even, the same on every rank)."""
    import torch
    n = S.shape[0]
    uc, q0, q1 = dist_layout(n, P, col_block, rank)
    cols = owned_columns(n, P, col_block, rank)
    Sl = torch.zeros((max(uc, 1), n), dtype=S.dtype, device=S.device)
    if len(cols):
        Sl[:len(cols)] = S[torch.as_tensor(cols, device=S.device)]
    Ql = None
    if Q is not None:
        # every rank's Q_loc has ld = ceil(n/P) (the last row block may be shorter)
        qld = -(-n // P)
        qld += qld & 1          # even: 16-byte aligned rows (TMA-describable)
        Ql = torch.zeros((n, max(2, qld)), dtype=Q.dtype, device=Q.device)
        Ql[:, :q1 - q0] = Q[:, q0:q1]
    return Sl, Ql


def unshard(S_locs, Q_locs, n: int, P: int, col_block: int):
    """Inverse of shard() over all ranks (numpy, column-major matrices as 2-D arrays)."""
    S = np.zeros((n, n))
    Q = None if Q_locs is None else np.zeros((n, n))
    for r in range(P):
        cols = owned_columns(n, P, col_block, r)
        Sl = S_locs[r].cpu().numpy() if hasattr(S_locs[r], "cpu") else S_locs[r]
        S[:, cols] = Sl[:len(cols)].T
        if Q is not None:
            _, q0, q1 = dist_layout(n, P, col_block, r)
            Ql = Q_locs[r].cpu().numpy() if hasattr(Q_locs[r], "cpu") else Q_locs[r]
            Q[q0:q1, :] = Ql.T[:q1 - q0]
    return S, Q


def reorder_dist_local(S_locs, Q_locs, select, n: int, col_block: int, window: int = 256, stream=None, **opts):
    """The sharded program for len(S_locs) ranks whose shards all live on the current device
    (sn_reorder_schur_dist_local).  Shards as produced by shard(); modified in place."""
    import torch
    P = len(S_locs)
    sp = (C.c_void_p * P)(*[C.c_void_p(t.data_ptr()) for t in S_locs])
    qp = None if Q_locs is None else (C.c_void_p * P)(*[C.c_void_p(t.data_ptr()) for t in Q_locs])
    ldq = 1
    if Q_locs is not None:
        ldq = max(1, max(t.shape[1] for t in Q_locs))
        for t in Q_locs:
            assert t.shape[1] == ldq, "Q shards must share one leading dimension (see shard())"
    o = default_opts(window=window, **opts)
    sel = np.ascontiguousarray(select, np.int32).copy()
    bmap = np.zeros(n, np.int8)
    m = C.c_int64()
    st = Stats()
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    rc = lib().sn_reorder_schur_dist_local(C.byref(o), P, n, col_block, sp, n, qp, ldq,
                                           sel.ctypes.data_as(C.c_void_p), C.byref(m),
                                           bmap.ctypes.data_as(C.c_void_p), C.byref(st), C.c_void_p(stream))
    return {"rc": rc, "m": m.value, "select": sel, "bmap": bmap, "stats": st.to_dict()}


def dist_init(rank: int, world: int, device: int, broadcast_id=None):
    """Create the library's NCCL communicator.  broadcast_id(bytes) -> bytes shares rank 0's
    unique id (default: torch.distributed.broadcast_object_list on the default group)."""
    buf = (C.c_char * 128)()
    if rank == 0:
        rc = lib().sn_dist_unique_id(buf)
        if rc:
            raise RuntimeError("sn_dist_unique_id rc=%d (%s)" % (rc, strerror(rc)))
    raw = bytes(buf)
    if broadcast_id is None:
        import torch.distributed as dist
        obj = [raw]
        dist.broadcast_object_list(obj, src=0)
        raw = obj[0]
    else:
        raw = broadcast_id(raw)
    buf = (C.c_char * 128).from_buffer_copy(raw)
    rc = lib().sn_dist_init(rank, world, buf, device)
    if rc:
        raise RuntimeError("sn_dist_init rc=%d (%s)" % (rc, strerror(rc)))


def dist_finalize():
    lib().sn_dist_finalize()


def reorder_dist(S_loc, Q_loc, select, n: int, col_block: int, window: int = 256, stream=None, **opts):
    """This rank's part of the sharded reordering (sn_reorder_schur_dist; collective)."""
    import torch
    o = default_opts(window=window, **opts)
    sel = np.ascontiguousarray(select, np.int32).copy()
    bmap = np.zeros(n, np.int8)
    m = C.c_int64()
    st = Stats()
    ldq = 1 if Q_loc is None else max(1, Q_loc.shape[1])
    if stream is None and S_loc.is_cuda:
        stream = torch.cuda.current_stream(S_loc.device).cuda_stream
    rc = lib().sn_reorder_schur_dist(C.byref(o), n, col_block, C.c_void_p(S_loc.data_ptr()), n,
                                     None if Q_loc is None else C.c_void_p(Q_loc.data_ptr()), ldq,
                                     sel.ctypes.data_as(C.c_void_p), C.byref(m), bmap.ctypes.data_as(C.c_void_p),
                                     C.byref(st), None if stream is None else C.c_void_p(stream))
    return {"rc": rc, "m": m.value, "select": sel, "bmap": bmap, "stats": st.to_dict()}


def dist_program(bmap, selrow, w: int, col_block: int, P: int, rank: int) -> np.ndarray:
    """Host only: rank's sharded program as an (R, 8) int64 record array (sn_reorder.h)."""
    bmap = np.ascontiguousarray(bmap, np.int8)
    selrow = np.ascontiguousarray(selrow, np.int8)
    n = len(bmap)
    L = lib()
    cnt = L.sn_dist_program(n, bmap.ctypes.data_as(C.c_void_p), selrow.ctypes.data_as(C.c_void_p), w, col_block,
                            P, rank, 0, None)
    if cnt < 0:
        raise ValueError("sn_dist_program rc=%d" % cnt)
    rec = np.zeros((cnt, 8), np.int64)
    L.sn_dist_program(n, bmap.ctypes.data_as(C.c_void_p), selrow.ctypes.data_as(C.c_void_p), w, col_block, P, rank,
                      cnt, rec.ctypes.data_as(C.c_void_p))
    return rec
