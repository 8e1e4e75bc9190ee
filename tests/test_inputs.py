import numpy as np

from oracle import ttlab_oracle as O
from paper_2601_16734_b200 import inputs as I


def test_generator_deterministic_and_normal():
    a = I.normals(200000, 1, 2, 3)
    b = I.normals(200000, 1, 2, 3)
    assert np.array_equal(a, b)
    assert abs(a.mean()) < 0.01 and abs(a.std() - 1) < 0.01
    assert not np.array_equal(a[:100], I.normals(100, 1, 2, 4))


def test_profiles_and_normalisation():
    assert I.bond_profile(6, 2, 5) == [1, 2, 4, 5, 4, 2, 1]
    ts = I.random_mps(12, 2, 16, 3)
    assert abs(O.MPS(ts).norm() - 1) < 1e-13
    ts = I.random_mps(8, 2, 4, 3, complex_=True)
    assert np.iscomplexobj(ts[0]) and abs(O.MPS(ts).norm() - 1) < 1e-13


def test_laplacian_is_periodic_second_difference():
    for n in range(2, 9):
        M = O.mpo_to_dense(O.MPO(I.laplacian_mpo(n))).real
        N = 2 ** n
        ref = -2 * np.eye(N) + np.roll(np.eye(N), 1, axis=1) + np.roll(np.eye(N), -1, axis=1)
        assert np.abs(M - ref).max() == 0.0
        S = O.mpo_to_dense(O.shift_mpo(n, 1)) + O.mpo_to_dense(O.shift_mpo(n, -1)) - 2 * np.eye(N)
        assert np.abs(S - M).max() == 0.0
    W = I.laplacian_mpo(20)
    assert [t.shape[0] for t in W] == [1] + [3] * 19
    assert set(np.unique(np.concatenate([t.ravel() for t in W]))) <= {-2.0, 0.0, 1.0}


def test_config4_mpo_bonds():
    W = I.random_mpo(30, 2, 8, 406)
    assert [t.shape[0] for t in W][:4] == [1, 4, 8, 8]
