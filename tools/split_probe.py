"""Per-kernel cost of one truncated split (preconditioner QRs + Jacobi) on single
matrices: kernel times (CUDA events) and Jacobi sweeps, raw vs preconditioned.
Usage: python tools/split_probe.py [reps]"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_16734_b200._lib import lib  # noqa: E402

REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 5
QR_KIND = int(__import__("os").environ.get("QR_KIND", "1"))  # 1 qr_small, 0 unblocked


def svd(th, mode=0):
    m, n = th.shape
    th = np.ascontiguousarray(th)
    iso = np.empty(max(m, n) ** 2)
    sv = np.empty(min(m, n))
    r, e2, sw, ms = C.c_int(), C.c_double(), C.c_int(), C.c_double()
    best = 1e9
    for _ in range(REPS):
        st = lib.ttg_debug_svd_ex(0, m, n, C.c_void_p(th.ctypes.data), mode, 1e-12, 0, C.c_void_p(iso.ctypes.data),
                                  sv.ctypes.data_as(C.POINTER(C.c_double)), C.byref(r), C.byref(e2), C.byref(sw),
                                  C.byref(ms), 0.0)
        assert st == 0, st
        best = min(best, ms.value * 1e3)
    ref = np.linalg.svd(th, compute_uv=False)
    return sw.value, best, np.linalg.norm(sv - ref) / np.linalg.norm(ref)


def qr_pre(A, withq):
    m, n = A.shape
    A = np.ascontiguousarray(A)
    k = min(m, n)
    Q = np.empty((m, k))
    RH = np.empty((n, k))
    ms = C.c_double()
    best = 1e9
    for _ in range(REPS):
        st = lib.ttg_debug_qr_pre(0, m, n, 0, C.c_void_p(A.ctypes.data), C.c_void_p(Q.ctypes.data) if withq else None,
                                  C.c_void_p(RH.ctypes.data), QR_KIND, C.byref(ms))
        assert st == 0, st
        best = min(best, ms.value * 1e3)
    return best


rng = np.random.default_rng(7)
import os
for n in [int(x) for x in os.environ.get("SIZES", "32,64,128").split(",")]:
    for decay in [float(x) for x in os.environ.get("DECAYS", "0,16").split(",")]:
        A = rng.standard_normal((n, n))
        if decay:
            U, _ = np.linalg.qr(rng.standard_normal((n, n)))
            V, _ = np.linalg.qr(rng.standard_normal((n, n)))
            A = (U * np.exp(-np.arange(n) / decay)) @ V.T
        _, R1 = np.linalg.qr(A)
        _, R2 = np.linalg.qr(R1.T)
        L = R2.T
        tq = qr_pre(A, True)
        tr = qr_pre(A, False)
        sr = svd(A)
        sl = svd(L)
        print(f"{n}x{n} decay={decay:4.0f}: qr+Q {tq:7.1f} us  qr(R) {tr:7.1f} us | jacobi raw {sr[0]:2d} sw "
              f"{sr[1]:7.1f} us (err {sr[2]:.1e}) | jacobi on L {sl[0]:2d} sw {sl[1]:7.1f} us (err {sl[2]:.1e}) | "
              f"split total ~{tq + tr + sl[1]:7.1f} us", flush=True)
