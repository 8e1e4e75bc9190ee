"""QFT through apply(MPOList) on the device (qft.hpp:107-112; test_lapack.cpp:265-335)."""
import numpy as np
import pytest

from oracle import ttlab_oracle as O

from ._compare import dense

pytestmark = pytest.mark.gpu


def _mods():
    from paper_2601_16734_b200 import qft as Q
    from paper_2601_16734_b200 import ttlab
    return Q, ttlab


def test_qft_reference_cases():
    Q, t = _mods()
    f = Q.qft(O.basis_state(6, 2, 0).tensors)
    assert np.abs(dense(f.to_tensors()) - 1.0 / 8.0).max() < 1e-12
    v = O.random_uniform_mps(6, 2, 3, 23)
    back = Q.iqft(Q.qft(v.tensors))
    assert np.linalg.norm(dense(back.to_tensors()) - O.mps_to_dense(v)) < 1e-12 * v.norm()
    v = O.random_uniform_mps(6, 2, 3, 24)
    x = O.mps_to_dense(v)
    got = dense(Q.qft_flip(Q.qft(v.tensors)).to_tensors())
    assert np.linalg.norm(got - np.fft.fft(x) / 8.0) < 1e-10
    # negative frequency lands at dim - 3: exp(-2 pi i 3 x / 64) is a product state
    ts = []
    for q in range(6):
        w = 2 ** (5 - q)
        ts.append(np.array([1.0, np.exp(-2j * np.pi * 3 * w / 64)]).reshape(1, 2, 1))
    f = dense(Q.qft_flip(Q.qft(ts)).to_tensors())
    assert int(np.argmax(np.abs(f))) == 64 - 3
    # subset transform on qubits {0, 1}
    v = O.random_uniform_mps(4, 2, 3, 26)
    out = t.apply(Q.qft_mpo(4, False, [0, 1]), v.tensors)
    assert np.linalg.norm(dense(out.to_tensors()) - O.qft_dense(4, sites=[0, 1]) @ O.mps_to_dense(v)) < 1e-10


def test_qft_large_smooth_function_against_fft():
    """L = 14 (16384 points): a Gaussian sampled on the grid has a low-rank MPS
    and so does its transform; compare with numpy's FFT."""
    Q, t = _mods()
    L = 14
    x = np.linspace(-1.0, 1.0, 1 << L, endpoint=False)
    g = np.exp(-x ** 2 / 0.02)
    g = g / np.linalg.norm(g)
    # exact MPS of the samples by successive SVDs (test-side helper)
    ts, rest, left = [], g.reshape(1, -1).astype(np.complex128), 1
    for k in range(L - 1):
        m = rest.reshape(left * 2, -1)
        u, s, vh = np.linalg.svd(m, full_matrices=False)
        r = max(1, int(np.sum(s > 1e-14 * s[0])))
        ts.append(u[:, :r].reshape(left, 2, r))
        rest = s[:r, None] * vh[:r]
        left = r
    ts.append(rest.reshape(left, 2, 1))
    strat = t.DEFAULT_STRATEGY.with_tolerance(1e-14)
    f = Q.qft_flip(Q.qft(ts, strat))
    got = dense(f.to_tensors())
    ref = np.fft.fft(g) / np.sqrt(1 << L)
    assert np.linalg.norm(got - ref) < 1e-9
    assert f.max_bond_dimension() <= 64
