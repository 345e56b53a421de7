"""Debug: the tiny problem of dbg_small.py through the raw C ABI in a process WITHOUT torch."""
import ctypes as C
import os
import sys

import numpy as np

d = np.load(sys.argv[1])
S = np.asfortranarray(d["S"]); Q = np.asfortranarray(d["Q"]); sel = d["sel"].astype(np.int32)
L = C.CDLL(os.path.join(os.getcwd(), "paper_1905_04975_b200", "libsn_b200.so"))
n = S.shape[0]
m = C.c_int64()
L.sn_reorder_schur.argtypes = [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(C.c_int64)]
rc = L.sn_reorder_schur(n, S.ctypes.data, n, Q.ctypes.data, n, sel.ctypes.data, C.byref(m))
print("notorch rc", rc, "m", m.value)
