"""Does a nearly-orthogonal start cut the Jacobi sweeps? (diagnostic)"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_16734_b200._lib import lib  # noqa: E402


def sweeps(th, mode=0):
    m, n = th.shape
    th = np.ascontiguousarray(th)
    iso = np.empty(max(m, n) ** 2)
    sv = np.empty(min(m, n))
    r, e2, sw, ms = C.c_int(), C.c_double(), C.c_int(), C.c_double()
    lib.ttg_debug_svd_ex(0, m, n, C.c_void_p(th.ctypes.data), mode, 1e-12, 0, C.c_void_p(iso.ctypes.data),
                         sv.ctypes.data_as(C.POINTER(C.c_double)), C.byref(r), C.byref(e2), C.byref(sw), C.byref(ms), 0.0)
    return sw.value, ms.value


rng = np.random.default_rng(1)
n = 128
U, _ = np.linalg.qr(rng.standard_normal((n, n)))
V, _ = np.linalg.qr(rng.standard_normal((n, n)))
for decay in (0.0, 1 / 16, 1 / 8, 1 / 4):
    s = np.exp(-decay * np.arange(n))
    th = (U * s) @ V.T
    print(f"decay {decay}: cold {sweeps(th)}", end="")
    print(f" | exact frame {sweeps(th @ V)}", end="")
    for eps in (1e-8, 1e-4, 1e-2):
        Vp, _ = np.linalg.qr(V + eps * rng.standard_normal((n, n)))
        print(f" | pert {eps:g}: {sweeps(th @ Vp)}", end="")
    print()

import scipy.linalg  # noqa: E402
print("QR preconditioning:")
for decay in (0.0, 1 / 16, 1 / 8, 1 / 4):
    s = np.exp(-decay * np.arange(n))
    th = (U * s) @ V.T
    q, r, piv = scipy.linalg.qr(th, pivoting=True)
    q2, r2 = np.linalg.qr(th)
    # R^T columns (Drmac-Veselic), R columns, unpivoted R^T
    print(f"decay {decay}: cold {sweeps(th)[0]} | piv R^T {sweeps(np.ascontiguousarray(r.T))[0]} "
          f"| piv R {sweeps(r)[0]} | unpiv R^T {sweeps(np.ascontiguousarray(r2.T))[0]} | th^T {sweeps(np.ascontiguousarray(th.T))[0]}")
print("double QR (Jacobi on L from R = L Q2):")
for decay in (1 / 16, 1 / 8, 1 / 4, 1 / 2):
    s = np.exp(-decay * np.arange(n))
    th = (U * s) @ V.T
    q, r, piv = scipy.linalg.qr(th, pivoting=True)
    Lp = np.ascontiguousarray(np.linalg.qr(r.T)[1].T)
    q2, r2 = np.linalg.qr(th)
    Lu = np.ascontiguousarray(np.linalg.qr(r2.T)[1].T)
    print(f"decay {decay}: cold {sweeps(th)[0]} | pivoted L {sweeps(Lp)[0]} | unpivoted L {sweeps(Lu)[0]} "
          f"| unpiv R {sweeps(r2)[0]}")
