"""Time the split preconditioner kernels (blocked qr_small vs unblocked) on one matrix."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_16734_b200._lib import lib  # noqa: E402

for (m, n) in [(128, 128), (64, 64), (256, 64), (96, 96)]:
    A = np.ascontiguousarray(np.random.default_rng(1).standard_normal((m, n)))
    k = min(m, n)
    Q = np.empty((m, k))
    RH = np.empty((n, k))
    for small in (1, 0):
        for withq in (1, 0):
            ts = []
            for _ in range(5):
                ms = C.c_double()
                lib.ttg_debug_qr_pre(0, m, n, 0, C.c_void_p(A.ctypes.data), C.c_void_p(Q.ctypes.data) if withq else None,
                                     C.c_void_p(RH.ctypes.data), small, C.byref(ms))
                ts.append(ms.value * 1e3)
            print(f"{m}x{n} small={small} Q={withq}: {min(ts):8.1f} us")
