"""Sweeps / time of the Jacobi SVD kernel for a few shapes and rotation thresholds."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_16734_b200._lib import lib  # noqa: E402


def run(th, mode, tol_rot):
    m, n = th.shape
    th = np.ascontiguousarray(th)
    iso = np.empty(max(m, n) ** 2)
    sv = np.empty(min(m, n))
    r, e2, sw, ms = C.c_int(), C.c_double(), C.c_int(), C.c_double()
    st = lib.ttg_debug_svd_ex(0, m, n, C.c_void_p(th.ctypes.data), mode, 1e-12, 0, C.c_void_p(iso.ctypes.data),
                              sv.ctypes.data_as(C.POINTER(C.c_double)), C.byref(r), C.byref(e2), C.byref(sw),
                              C.byref(ms), tol_rot)
    ref = np.linalg.svd(th, compute_uv=False)
    return st, sw.value, ms.value, np.abs(sv - ref).max() / ref[0]


rng = np.random.default_rng(0)
if len(sys.argv) > 1:
    m = n = int(sys.argv[1])
    A = rng.standard_normal((m, n))
    if len(sys.argv) > 2:  # graded spectrum exp(-k/decay)
        U, _ = np.linalg.qr(rng.standard_normal((m, m)))
        V, _ = np.linalg.qr(rng.standard_normal((n, n)))
        A = (U * np.exp(-np.arange(m) / float(sys.argv[2]))) @ V.T
    run(A, 0, 0.0)  # warm-up (module load, smem attribute)
    print(run(A, 0, 0.0), run(A, 1, 0.0))
    sys.exit(0)
for (m, n) in [(32, 32), (64, 64), (128, 128), (192, 128), (128, 192), (256, 256)]:
    for decay in (False, True):
        A = rng.standard_normal((m, n))
        if decay:
            U, _ = np.linalg.qr(rng.standard_normal((m, m)))
            V, _ = np.linalg.qr(rng.standard_normal((n, n)))
            k = min(m, n)
            s = np.exp(-np.arange(k) / 8.0)
            A = (U[:, :k] * s) @ V[:, :k].T
        for mode in (0, 1):
            for tr in (0.0, np.sqrt(max(m, n)) * 2.2e-16, 1e-13):
                st, sw, ms, err = run(A, mode, tr)
                print(f"{m}x{n} decay={int(decay)} mode={mode} tol_rot={tr:.1e}: st={st} sweeps={sw} "
                      f"{ms * 1e3:8.1f} us  max|ds|/s0={err:.1e}", flush=True)
