"""Blocked QR timing on one matrix (diagnostic): python tools/qr_probe.py m n [c]"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2601_16734_b200._lib import lib  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
cplx = len(sys.argv) > 3
dt = np.complex128 if cplx else np.float64
A = np.random.default_rng(0).standard_normal((m, n)).astype(dt)
k = min(m, n)
Q = np.empty((m, k), dtype=dt)
R = np.empty((k, n), dtype=dt)
for _ in range(2):
    t = time.time()
    st = lib.ttg_debug_qr_blocked(1 if cplx else 0, m, n, C.c_void_p(A.ctypes.data), C.c_void_p(Q.ctypes.data),
                                  C.c_void_p(R.ctypes.data))
    print(st, f"{(time.time() - t) * 1e3:.1f} ms (incl. H2D/D2H)", np.abs(Q @ R - A).max())
