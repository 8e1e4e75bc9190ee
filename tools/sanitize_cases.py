"""Smallest cases that launch the kernels with cross-thread / cross-CTA synchronisation, for
compute-sanitizer (racecheck / synccheck), one tool per run:
  jacobi_cluster_kernel (DSMEM ring + cluster barrier), jacobi_wp_kernel and jacobi_grid_kernel
  (cooperative grid barriers), iso_complete_kernel, qr_panel_cl_kernel (cluster panel), t_combine_kernel
  (two-level blocked QR), split-K gemm_kernel + splitk_reduce_kernel, and one small apply+simplify
  through the engine.  Usage: compute-sanitizer --tool racecheck python tools/sanitize_cases.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_16734_b200._lib import lib  # noqa: E402


def svd(th, mode=0, tol=1e-12):
    m, n = th.shape
    th = np.ascontiguousarray(th)
    iso = np.empty(max(m, n) ** 2)
    sv = np.empty(min(m, n))
    r, e2 = C.c_int(), C.c_double()
    st = lib.ttg_debug_svd(0, m, n, C.c_void_p(th.ctypes.data), mode, tol, 0, C.c_void_p(iso.ctypes.data),
                           sv.ctypes.data_as(C.POINTER(C.c_double)), C.byref(r), C.byref(e2))
    assert st == 0, st
    return sv


def qr_blocked(m, n):
    a = np.random.default_rng(m + n).standard_normal((m, n))
    k = min(m, n)
    q, r = np.empty(m * k), np.empty(k * n)
    assert lib.ttg_debug_qr_blocked(0, m, n, C.c_void_p(a.ctypes.data), C.c_void_p(q.ctypes.data),
                                    C.c_void_p(r.ctypes.data)) == 0
    assert np.abs(q.reshape(m, k) @ r.reshape(k, n) - a).max() < 1e-10


rng = np.random.default_rng(0)
which = sys.argv[1:] or ["cluster", "grid", "wp", "complete", "qr", "splitk", "engine"]
if "cluster" in which:  # single-chain 65..128-column split -> jacobi_cluster_kernel
    svd(rng.standard_normal((96, 96)))
if "wp" in which or "grid" in which:
    os.environ["TTG_DEBUG_SVD_GRID"] = "1"  # read per call by the debug hook
    svd(rng.standard_normal((256, 200)))  # warp-pair grid kernel (default)
if "complete" in which:  # kept numerically-zero values -> iso_complete_kernel
    a = rng.standard_normal((48, 10)) @ rng.standard_normal((10, 40))
    svd(a, 0, 0.0)
if "qr" in which:
    qr_blocked(2048, 64)    # cluster panels (qr_panel_cl_kernel)
    qr_blocked(640, 520)    # two-level: t_combine_kernel + K = 128 updates
if "splitk" in which:  # few output tiles, long K -> split-K partials + ordered reduction
    M, N, K = 32, 64, 4096
    A, B = rng.standard_normal((M, K)), rng.standard_normal((K, N))
    Cm = np.empty((M, N))
    assert lib.ttg_debug_gemm(0, 0, 0, M, N, K, 1, C.c_void_p(A.ctypes.data), C.c_void_p(B.ctypes.data),
                              C.c_void_p(Cm.ctypes.data)) == 0
    assert np.abs(Cm - A @ B).max() < 1e-10
if "engine" in which:
    from paper_2601_16734_b200 import inputs as I
    from paper_2601_16734_b200 import ttlab
    psi = I.random_mps(10, 2, 16, 3)
    W = I.laplacian_mpo(10)
    out = ttlab.apply(W, psi, ttlab.Strategy(max_bond=16, max_sweeps=2))
    assert max(out.bond_dimensions()) <= 16
print("SANITIZE_CASES_OK", which)
