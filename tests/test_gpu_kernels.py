"""Kernel-level parity: DMMA GEMM, Householder QR and the truncated Jacobi SVD
against numpy, through the C-ABI test hooks of libttgpu.so."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OPS = {0: lambda x: x, 1: lambda x: x.T, 2: lambda x: x.conj().T, 3: lambda x: x.conj()}


def _lib():
    from paper_2601_16734_b200._lib import lib
    return lib


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


def _gemm(opA, opB, A, B, M, N, K, batch):
    lib = _lib()
    cplx = np.iscomplexobj(A)
    Cm = np.empty((batch, M, N), dtype=A.dtype)
    st = lib.ttg_debug_gemm(1 if cplx else 0, opA, opB, M, N, K, batch, _ptr(A), _ptr(B), _ptr(Cm))
    assert st == 0
    return Cm


@pytest.mark.parametrize("dtype", [np.float64, np.complex128])
@pytest.mark.parametrize("opA", [0, 1, 2, 3])
@pytest.mark.parametrize("opB", [0, 1, 2, 3])
def test_gemm_ops(dtype, opA, opB):
    rng = np.random.default_rng(opA * 4 + opB)
    for (M, N, K) in [(1, 1, 1), (5, 7, 3), (64, 64, 16), (65, 130, 17), (128, 96, 200), (3, 190, 1)]:
        batch = 2

        def rnd(*s):
            x = rng.standard_normal(s)
            if dtype == np.complex128:
                x = x + 1j * rng.standard_normal(s)
            return x

        Ash = (batch, M, K) if opA in (0, 3) else (batch, K, M)
        Bsh = (batch, K, N) if opB in (0, 3) else (batch, N, K)
        A, B = np.ascontiguousarray(rnd(*Ash)), np.ascontiguousarray(rnd(*Bsh))
        got = _gemm(opA, opB, A, B, M, N, K, batch)
        for b in range(batch):
            ref = OPS[opA](A[b]) @ OPS[opB](B[b])
            err = np.abs(got[b] - ref).max() / max(1.0, np.abs(ref).max())
            assert err < 1e-13, (M, N, K, err)


_TMA_SNIPPET = """
import sys
import numpy as np
sys.path.insert(0, '.')
from tests.test_gpu_kernels import OPS, _gemm
worst = 0.0
for dtype in (np.float64, np.complex128):
    for opA in range(4):
        for opB in range(4):
            rng = np.random.default_rng(16 * opA + opB)
            for (M, N, K, batch) in [(128, 96, 192, 2), (64, 190, 64, 2), (200, 130, 256, 1), (70, 66, 1024, 1),
                                     (64, 64, 40, 1), (130, 258, 72, 1), (512, 320, 272, 1)]:
                def rnd(*s):
                    x = rng.standard_normal(s)
                    return x + 1j * rng.standard_normal(s) if dtype == np.complex128 else x
                Ash = (batch, M, K) if opA in (0, 3) else (batch, K, M)
                Bsh = (batch, K, N) if opB in (0, 3) else (batch, N, K)
                A, B = np.ascontiguousarray(rnd(*Ash)), np.ascontiguousarray(rnd(*Bsh))
                got = _gemm(opA, opB, A, B, M, N, K, batch)
                for b in range(batch):
                    ref = OPS[opA](A[b]) @ OPS[opB](B[b])
                    worst = max(worst, np.abs(got[b] - ref).max() / max(1.0, np.abs(ref).max()))
assert worst < 1e-13, worst
print('TMA_GEMM_OK', worst)
"""


def test_gemm_tma_all_ops():
    """The TMA-staged GEMM variants for every operand mode and both dtypes: bulk row copies + mbarrier
    pipeline (TTG_GEMM_TMA=2 routes all eligible products to it; by default only m-/n-contiguous operand
    pairs use it) and, for single-chain f64 products with A = N and B = N / T, the tensor-map kernel
    (cp.async.bulk.tensor, swizzled tiles; TTG_GEMM_TM=2 lifts its size threshold), including split-K
    (K = 1024 with few tiles), ragged K and partial edge tiles."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TTG_GEMM_TMA="2", TTG_GEMM_TM="2")
    r = subprocess.run([sys.executable, "-c", _TMA_SNIPPET], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "TMA_GEMM_OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("blocked", [False, True])
@pytest.mark.parametrize("dtype", [np.float64, np.complex128])
@pytest.mark.parametrize("shape", [(1, 1), (2, 3), (8, 4), (4, 8), (64, 32), (130, 70), (384, 192), (96, 200),
                                   (1000, 300), (257, 65), (4100, 70), (8192, 40), (2048, 300), (1100, 600),
                                   (700, 700), (600, 1030), (6000, 130)])
def test_householder_qr(dtype, shape, blocked):
    lib = _lib()
    m, n = shape
    k = min(m, n)
    rng = np.random.default_rng(m * 1000 + n)
    A = rng.standard_normal((m, n))
    if dtype == np.complex128:
        A = A + 1j * rng.standard_normal((m, n))
    A = np.ascontiguousarray(A)
    Q = np.empty((m, k), dtype=dtype)
    R = np.empty((k, n), dtype=dtype)
    fn = lib.ttg_debug_qr_blocked if blocked else lib.ttg_debug_qr
    assert fn(1 if dtype == np.complex128 else 0, m, n, _ptr(A), _ptr(Q), _ptr(R)) == 0
    assert np.abs(Q.conj().T @ Q - np.eye(k)).max() < 1e-13
    assert np.abs(Q @ R - A).max() < 1e-12 * max(1, np.abs(A).max())
    assert np.abs(np.tril(R, -1)).max() == 0.0


def test_qr_rank_deficient():
    lib = _lib()
    rng = np.random.default_rng(5)
    A = np.ascontiguousarray(rng.standard_normal((40, 3)) @ rng.standard_normal((3, 20)))
    Q, R = np.empty((20, 20))[:0], None
    Q = np.empty((40, 20))
    R = np.empty((20, 20))
    for fn in (lib.ttg_debug_qr, lib.ttg_debug_qr_blocked):
        assert fn(0, 40, 20, _ptr(A), _ptr(Q), _ptr(R)) == 0
        assert np.abs(Q.T @ Q - np.eye(20)).max() < 1e-13
        assert np.abs(Q @ R - A).max() < 1e-12 * np.abs(A).max()


def _svd(theta, mode, tol=0.0, max_bond=0):
    lib = _lib()
    m, n = theta.shape
    cplx = np.iscomplexobj(theta)
    theta = np.ascontiguousarray(theta)
    iso = np.empty(max(m, n) * max(m, n), dtype=theta.dtype)
    sv = np.empty(min(m, n))
    r, e2 = C.c_int(), C.c_double()
    st = lib.ttg_debug_svd(1 if cplx else 0, m, n, _ptr(theta), mode, tol, max_bond, _ptr(iso),
                           sv.ctypes.data_as(C.POINTER(C.c_double)), C.byref(r), C.byref(e2))
    assert st == 0
    r = r.value
    iso = iso[:m * r].reshape(m, r) if mode == 0 else iso[:r * n].reshape(r, n)
    return iso, sv, r, e2.value


@pytest.fixture(params=["cta", "grid"])
def svd_impl(request, monkeypatch):
    monkeypatch.setenv("TTG_DEBUG_SVD_GRID", "1" if request.param == "grid" else "0")
    return request.param


@pytest.mark.parametrize("dtype", [np.float64, np.complex128])
@pytest.mark.parametrize("shape", [(1, 1), (2, 2), (4, 4), (6, 4), (4, 6), (32, 32), (128, 128), (64, 150), (192, 128),
                                   (300, 260)])
@pytest.mark.parametrize("mode", [0, 1])
def test_jacobi_svd_random(dtype, shape, mode, svd_impl):
    m, n = shape
    rng = np.random.default_rng(m * 7 + n)
    th = rng.standard_normal((m, n))
    if dtype == np.complex128:
        th = th + 1j * rng.standard_normal((m, n))
    iso, sv, r, e2 = _svd(th, mode)
    ref = np.linalg.svd(th, compute_uv=False)
    assert np.abs(sv - ref).max() <= 1e-13 * ref[0]
    assert r == min(m, n)
    if mode == 0:
        assert np.abs(iso.conj().T @ iso - np.eye(r)).max() < 1e-12
        # U_r U_r^H theta == theta (full rank kept)
        assert np.abs(iso @ (iso.conj().T @ th) - th).max() < 1e-12 * ref[0]
    else:
        assert np.abs(iso @ iso.conj().T - np.eye(r)).max() < 1e-12
        assert np.abs((th @ iso.conj().T) @ iso - th).max() < 1e-12 * ref[0]


@pytest.mark.parametrize("dtype,shape", [(np.float64, (600, 520)), (np.float64, (1000, 700)), (np.float64, (1024, 1024)),
                                         (np.float64, (1536, 1536)), (np.float64, (2048, 1100)),
                                         (np.complex128, (480, 300)), (np.complex128, (300, 480)),
                                         (np.complex128, (1000, 520))])
@pytest.mark.parametrize("mode", [0, 1])
def test_jacobi_svd_grid_large(dtype, shape, mode, monkeypatch):
    """Grid-cooperative block Jacobi at the C3/C4 split sizes (rows split over 2-CTA clusters)."""
    monkeypatch.setenv("TTG_DEBUG_SVD_GRID", "1")
    m, n = shape
    rng = np.random.default_rng(m + 3 * n)
    th = rng.standard_normal((m, n))
    if dtype == np.complex128:
        th = th + 1j * rng.standard_normal((m, n))
    iso, sv, r, e2 = _svd(th, mode)
    ref = np.linalg.svd(th, compute_uv=False)
    assert np.abs(sv - ref).max() <= 1e-12 * ref[0]
    assert r == min(m, n)
    if mode == 0:
        assert np.abs(iso.conj().T @ iso - np.eye(r)).max() < 1e-12
    else:
        assert np.abs(iso @ iso.conj().T - np.eye(r)).max() < 1e-12


def test_svd_kat_identity():
    """test_core.cpp:74-90: theta = I/sqrt(2)."""
    th = np.eye(2) / np.sqrt(2.0)
    iso, sv, r, e2 = _svd(th, 0)
    assert r == 2 and e2 == 0.0
    assert np.allclose(sv, [1 / np.sqrt(2)] * 2, rtol=0, atol=1e-15)
    iso, sv, r, e2 = _svd(th, 0, max_bond=1)
    assert r == 1 and abs(np.sqrt(e2) - 1 / np.sqrt(2)) < 1e-15


def test_svd_truncation_rule(svd_impl):
    """schmidt.hpp:40-59: strict > tol*s0, at least 1, at most max_bond; err = sqrt(sum dropped^2)."""
    rng = np.random.default_rng(3)
    U, _ = np.linalg.qr(rng.standard_normal((10, 10)))
    V, _ = np.linalg.qr(rng.standard_normal((10, 10)))
    s = np.array([1.0, 0.5, 0.25, 1e-3, 1e-6, 1e-9, 1e-11, 1e-13, 1e-15, 0.0])
    th = (U * s) @ V.T
    _, sv, r, e2 = _svd(th, 0, tol=1e-10)
    assert r == 6
    assert abs(np.sqrt(e2) - np.sqrt(np.sum(s[6:] ** 2))) < 1e-15
    _, sv, r, e2 = _svd(th, 1, tol=1e-10, max_bond=3)
    assert r == 3
    assert abs(np.sqrt(e2) - np.sqrt(np.sum(s[3:] ** 2))) < 1e-15
    _, _, r, _ = _svd(np.zeros((3, 3)), 0, tol=1e-10)
    assert r == 1


def test_svd_rank_deficient_drops_zero_values(svd_impl):
    rng = np.random.default_rng(11)
    th = rng.standard_normal((64, 5)) @ rng.standard_normal((5, 64))
    _, sv, r, _ = _svd(th, 0, tol=1e-12)
    assert r == 5
    assert sv[5] < 1e-12 * sv[0]


@pytest.mark.parametrize("dtype", [np.float64, np.complex128])
@pytest.mark.parametrize("shape,trans", [((128, 128), 0), ((128, 128), 1), ((64, 64), 0), ((100, 37), 0),
                                         ((37, 100), 1), ((200, 96), 0), ((24, 80), 0), ((250, 60), 0),
                                         ((17, 5), 1), ((128, 40), 1)])
def test_qr_precondition_small_kernel(dtype, shape, trans):
    """qr_small.cu (blocked, register panels) against the definition M = Q R and
    against the unblocked preconditioner it replaces."""
    lib = _lib()
    m, n = shape
    rng = np.random.default_rng(m * 7 + n)
    A = rng.standard_normal((m, n))
    if dtype == np.complex128:
        A = A + 1j * rng.standard_normal((m, n))
    A = np.ascontiguousarray(A)
    M = A.conj().T if trans else A
    l, k = M.shape
    r0 = min(l, k)
    code = 1 if dtype == np.complex128 else 0
    if 16 * l * k > 200 * 1024 and code == 1:
        pytest.skip("complex panel does not fit shared memory")
    out = {}
    for small in (1, 0):
        Q = np.empty((l, r0), dtype=dtype)
        RH = np.empty((k, r0), dtype=dtype)
        ms = C.c_double()
        assert lib.ttg_debug_qr_pre(code, m, n, trans, _ptr(A), _ptr(Q), _ptr(RH), small, C.byref(ms)) == 0
        R = RH.conj().T
        assert np.abs(Q.conj().T @ Q - np.eye(r0)).max() < 1e-13
        assert np.abs(Q @ R - M).max() < 1e-12 * np.abs(M).max()
        assert np.abs(np.tril(R, -1)).max() == 0.0
        out[small] = (Q, R)
        # R only (no Q)
        RH2 = np.empty((k, r0), dtype=dtype)
        assert lib.ttg_debug_qr_pre(code, m, n, trans, _ptr(A), None, _ptr(RH2), small, C.byref(ms)) == 0
        assert np.array_equal(RH2, RH)
    # same Householder convention: identical factors up to rounding
    assert np.abs(out[1][1] - out[0][1]).max() < 1e-12 * np.abs(M).max()


def test_qr_precondition_small_rank_deficient():
    lib = _lib()
    rng = np.random.default_rng(11)
    A = np.ascontiguousarray(rng.standard_normal((128, 5)) @ rng.standard_normal((5, 128)))
    Q = np.empty((128, 128))
    RH = np.empty((128, 128))
    assert lib.ttg_debug_qr_pre(0, 128, 128, 0, _ptr(A), _ptr(Q), _ptr(RH), 1, None) == 0
    assert np.abs(Q.T @ Q - np.eye(128)).max() < 1e-13
    assert np.abs(Q @ RH.T - A).max() < 1e-12 * np.abs(A).max()


@pytest.mark.parametrize("dtype", [np.float64, np.complex128])
@pytest.mark.parametrize("mode", [0, 1])
def test_svd_kept_negligible_values_orthonormal(dtype, mode, svd_impl):
    """tol = 0 (NO_TRUNCATION) keeps numerically-zero singular values; their vectors
    must still complete an orthonormal isometry (Eigen JacobiSVD semantics), so the
    split reconstructs theta."""
    rng = np.random.default_rng(21 + mode)
    m, n, rank = 64, 48, 20
    a, b = rng.standard_normal((m, rank)), rng.standard_normal((rank, n))
    if dtype == np.complex128:
        a = a + 1j * rng.standard_normal((m, rank))
    th = a @ b
    iso, sv, r, _ = _svd(th, mode, tol=0.0)
    assert rank < r <= min(m, n)  # roundoff values are kept (strict > 0 cutoff)
    assert sv[rank] < 1e-12 * sv[0]
    if mode == 0:
        assert np.abs(iso.conj().T @ iso - np.eye(r)).max() < 1e-12
        assert np.abs(iso @ (iso.conj().T @ th) - th).max() < 1e-12 * sv[0]
    else:
        assert np.abs(iso @ iso.conj().T - np.eye(r)).max() < 1e-12
        assert np.abs((th @ iso.conj().T) @ iso - th).max() < 1e-12 * sv[0]


@pytest.mark.parametrize("seed", [0, 4])
@pytest.mark.parametrize("n", [64, 128, 256])
def test_svd_clustered_spectrum_isometry(n, seed, svd_impl):
    """Near-degenerate Schmidt spectra (blocks sigma = 1 +- 1e-9): the early stop must
    not leave the isometry non-orthogonal.  n = 128 runs on the cluster kernel; seeds n and n + 4
    left 1.7e-12 / 2.6e-12 before the rotation-angle guard of the stop rule (sweep_stop)."""
    rng = np.random.default_rng(n + seed)
    U, _ = np.linalg.qr(rng.standard_normal((n, n)))
    V, _ = np.linalg.qr(rng.standard_normal((n, n)))
    s = np.repeat([1.0, 0.5, 0.1, 1e-3], n // 4) * (1 + 1e-9 * rng.standard_normal(n))
    th = (U * s) @ V.T
    for mode in (0, 1):
        iso, sv, r, _ = _svd(th, mode, tol=1e-12)
        if mode == 0:
            assert np.abs(iso.conj().T @ iso - np.eye(r)).max() < 1e-12
        else:
            assert np.abs(iso @ iso.conj().T - np.eye(r)).max() < 1e-12
        assert np.abs(sv - np.sort(s)[::-1]).max() < 1e-13


@pytest.mark.parametrize("shape", [(47, 6), (5, 64), (66, 9), (112, 113), (75, 258), (182, 147), (319, 141)])
@pytest.mark.parametrize("mode", [0, 1])
def test_svd_clustered_spectrum_isometry_complex(shape, mode):
    """Complex splits with clustered singular values (sigma = 1 +- 1e-9) on the shapes tools/fuzz_split.py
    caught: the register-blocked one-CTA kernel stopped early without the guards of the ring kernels and left
    |U^H U - I| up to 9e-10."""
    m, n = shape
    k = min(m, n)
    rng = np.random.default_rng(m * 1000 + n)
    U, _ = np.linalg.qr(rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k)))
    V, _ = np.linalg.qr(rng.standard_normal((n, k)) + 1j * rng.standard_normal((n, k)))
    s = np.sort(1.0 + 1e-9 * rng.standard_normal(k))[::-1]
    th = (U * s) @ V.conj().T
    iso, sv, r, _ = _svd(th, mode, tol=1e-12)
    assert r == k
    if mode == 0:
        assert np.abs(iso.conj().T @ iso - np.eye(r)).max() < 1e-12
        assert np.abs(iso @ (iso.conj().T @ th) - th).max() < 1e-11
    else:
        assert np.abs(iso @ iso.conj().T - np.eye(r)).max() < 1e-12
        assert np.abs((th @ iso.conj().T) @ iso - th).max() < 1e-11
    assert np.abs(sv - s).max() < 1e-13


_RETRY_SNIPPET = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from oracle import ttlab_oracle as O
from paper_2601_16734_b200 import inputs as I, ttlab
from tests._compare import dense, rel
psi = I.random_mps(12, 2, 32, 101)
strat = ttlab.Strategy(max_bond=12, max_sweeps=3)
rep = []
out = ttlab.simplify(psi, strat, report=rep)
rr = {}
ref = O.simplify(O.MPS(psi), O.Strategy(max_bond=12, max_sweeps=3), report=rr)
assert out.bond_dimensions() == ref.bond_dimensions()
assert rep[0]["sweeps"] == rr["sweeps"]
assert abs(rep[0]["residual"] - rr["residual"]) < 1e-10
assert rel(dense(out.to_tensors()), O.mps_to_dense(ref)) < 1e-10
print("RETRY_OK")
'''


def test_svd_forced_retry_matches_oracle():
    """schmidt.hpp:23-35: a split that fails its first attempt is jittered by
    1e-14 |theta| and retried.  TTG_SVD_FORCE_RETRY=1 caps the first attempt at one
    Jacobi sweep, so every split takes the retry path; the result must still match
    the oracle (the jitter is far below the 1e-10 parity tolerance)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TTG_SVD_FORCE_RETRY="1")
    r = subprocess.run([sys.executable, "-c", _RETRY_SNIPPET], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "RETRY_OK" in r.stdout, r.stdout + r.stderr
    env2 = dict(os.environ, TTG_SVD_FORCE_RETRY="1")
    snippet = ("import sys, numpy as np; sys.path.insert(0, '.'); from tests.test_gpu_kernels import _svd; "
               "th = np.random.default_rng(5).standard_normal((40, 40)); iso, sv, r, e2 = _svd(th, 0); "
               "ref = np.linalg.svd(th, compute_uv=False); assert np.abs(sv - ref).max() < 1e-12 * ref[0]; "
               "assert np.abs(iso.T @ iso - np.eye(r)).max() < 1e-12; print('SVD_RETRY_OK')")
    r = subprocess.run([sys.executable, "-c", snippet], cwd=root, env=env2, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "SVD_RETRY_OK" in r.stdout, r.stdout + r.stderr
