"""Grid Jacobi variants on C4-like split matrices: time, sweeps, accuracy.
Usage: TTG_SVD_WP=<0|4|8> TTG_DEBUG_SVD_GRID=1 python tools/wp_probe.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_16734_b200._lib import lib  # noqa: E402


def run(th, mode):
    m, n = th.shape
    cplx = np.iscomplexobj(th)
    th = np.ascontiguousarray(th)
    iso = np.empty(max(m, n) ** 2, dtype=th.dtype)
    sv = np.empty(min(m, n))
    r, e2, sw, ms = C.c_int(), C.c_double(), C.c_int(), C.c_double()
    st = lib.ttg_debug_svd_ex(1 if cplx else 0, m, n, C.c_void_p(th.ctypes.data), mode, 1e-12, 0,
                              C.c_void_p(iso.ctypes.data), sv.ctypes.data_as(C.POINTER(C.c_double)), C.byref(r),
                              C.byref(e2), C.byref(sw), C.byref(ms), 0.0)
    ref = np.linalg.svd(th, compute_uv=False)
    r = r.value
    U = iso[:m * r].reshape(m, r) if mode == 0 else iso[:r * n].reshape(r, n).conj().T
    orth = np.abs(U.conj().T @ U - np.eye(r)).max()
    return st, sw.value, ms.value, np.abs(sv - ref).max() / ref[0], orth


rng = np.random.default_rng(0)


def c4_like(m, n, cplx=False):
    k = min(m, n)
    U = np.linalg.qr(rng.standard_normal((m, k)))[0]
    V = np.linalg.qr(rng.standard_normal((n, k)))[0]
    s = np.exp(np.linspace(0, np.log(1e-5), k)) * (1 + 0.01 * rng.standard_normal(k))
    A = (U * s) @ V.T
    if cplx:
        A = A + 1j * ((U * s) @ np.linalg.qr(rng.standard_normal((n, k)))[0].T)
    return A


tag = os.environ.get("TTG_SVD_WP", "8")
for (m, n, cplx) in ([] if __name__ != "__main__" else [(1024, 1024, False), (512, 1024, False), (256, 256, True), (256, 512, True)]):
    A = c4_like(m, n, cplx)
    L = np.linalg.qr(np.linalg.qr(A)[1].conj().T)[1].conj().T  # Drmac-Veselic preconditioned matrix
    run(L, 0)
    for name, M in (("raw", A), ("precond", np.ascontiguousarray(L))):
        st, sw, ms, err, orth = run(M, 0 if name == "raw" else 0)
        print(f"WP={tag} {m}x{n} {'c128' if cplx else 'f64'} {name}: st={st} sweeps={sw} {ms:8.2f} ms "
              f"({ms / max(sw, 1):.3f} ms/sweep)  |ds|/s0={err:.1e} orth={orth:.1e}", flush=True)
