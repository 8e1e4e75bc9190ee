"""Two-site effective operator matvec (eigensolvers.hpp:15-64): the oracle restatement pinned to
the network identity <psi|H|psi> = x^H H_eff x (operator environments of environments.hpp:42-83
around sites (k, k+1)), and the device path against the oracle."""
import numpy as np
import pytest

from oracle import ttlab_oracle as O
from paper_2601_16734_b200 import inputs as I


def _case(n=6, k=2, chi=6, D=3, seed=7, cplx=True):
    rng = np.random.default_rng(seed)
    psi = O.MPS(I.random_mps(n, 2, chi, seed, complex_=cplx))
    mpo = O.MPO(I.laplacian_mpo(n)) if D == 3 else None
    if mpo is None:
        ws = []
        for i in range(n):
            l = 1 if i == 0 else D
            r = 1 if i == n - 1 else D
            ws.append(rng.standard_normal((l, 2, 2, r)) + (1j * rng.standard_normal((l, 2, 2, r)) if cplx else 0))
        mpo = O.MPO(ws)
    L = np.ones((1, 1, 1), dtype=np.complex128)
    for i in range(k):
        L = O.update_left_op_environment(L, psi[i], mpo[i], psi[i])
    R = np.ones((1, 1, 1), dtype=np.complex128)
    for i in range(n - 1, k + 1, -1):
        R = O.update_right_op_environment(R, psi[i], mpo[i], psi[i])
    x = np.einsum("asb,btc->astc", psi[k], psi[k + 1]).reshape(-1)
    return psi, mpo, L, R, x, k


@pytest.mark.parametrize("D", [3, 4])
def test_oracle_heff_network_identity(D):
    psi, mpo, L, R, x, k = _case(D=D)
    # L is E[c](a, b) with a the bra bond: the matvec's lenv[c0](a', a) = E[c0](a', a)
    y = O.apply_effective_two_site(L, mpo[k], mpo[k + 1], R, x)
    ref = O.expectation_mpo(mpo, psi)
    assert abs(np.vdot(x, y) - ref) <= 1e-12 * max(1.0, abs(ref))


def test_oracle_heff_bad_size():
    psi, mpo, L, R, x, k = _case()
    with pytest.raises(O.ShapeError):
        O.apply_effective_two_site(L, mpo[k], mpo[k + 1], R, x[:-1])


@pytest.mark.gpu
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("D,chi", [(3, 6), (4, 16), (8, 40)])
def test_gpu_heff_matches_oracle(cplx, D, chi):
    from paper_2601_16734_b200 import ttlab as t
    psi, mpo, L, R, x, k = _case(n=8, k=3, chi=chi, D=D, cplx=cplx)
    if not cplx:
        L, R = L.real.copy(), R.real.copy()
    w1 = mpo[k] if cplx else np.real(mpo[k])
    w2 = mpo[k + 1] if cplx else np.real(mpo[k + 1])
    xx = x if cplx else x.real
    y = t.apply_effective_two_site(L, w1, w2, R, xx)
    ref = O.apply_effective_two_site(L, w1, w2, R, xx)
    assert y.shape == ref.shape
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.gpu
def test_gpu_heff_shape_errors():
    from paper_2601_16734_b200 import ttlab as t
    psi, mpo, L, R, x, k = _case()
    with pytest.raises(t.ShapeError):
        t.apply_effective_two_site(L, mpo[k], mpo[k + 1], R, x[:-1])
    with pytest.raises(t.ShapeError):
        bad = np.ones((mpo[k].shape[3] + 1, 2, 2, mpo[k + 1].shape[3]))  # w2 left bond != w1 right bond
        t.apply_effective_two_site(L, mpo[k], bad, R, x)
