"""QFT layers (qft.hpp:10-128): the oracle's dense circuit pinned against the
reference's qft test cases (test_lapack.cpp:265-335), and the product's host
MPO constructors checked layer by layer against it (no GPU needed)."""
import numpy as np
import pytest

from oracle import ttlab_oracle as O


def _dft(L):
    dim = 1 << L
    j = np.arange(dim)
    return np.exp(-2j * np.pi * np.outer(j, j) / dim) / np.sqrt(dim)


def test_oracle_qft_pins():
    L = 6
    U = O.qft_dense(L)
    e0 = np.zeros(1 << L)
    e0[0] = 1.0
    assert np.abs(U @ e0 - 1.0 / 8.0).max() < 1e-12  # test_lapack.cpp:266-271
    assert np.abs(O.bit_reversal(L) @ U - _dft(L)).max() < 1e-12  # :278-291
    assert np.abs(O.qft_dense(L, inverse=True) @ U - np.eye(1 << L)).max() < 1e-12  # :273-276
    for m in range(5):  # :293-299
        Lm = O.qft_layer_dense(5, list(range(5)), m, -1.0, False)
        assert np.linalg.norm(Lm.conj().T @ Lm - np.eye(32)) < 1e-12
    # negative frequency -> index dim - 3 (:300-311)
    x = np.arange(64)
    f = O.bit_reversal(L) @ U @ np.exp(-2j * np.pi * 3 * x / 64)
    assert int(np.argmax(np.abs(f))) == 64 - 3
    # subset transform (:318-334)
    dft4 = np.exp(-2j * np.pi * np.outer(np.arange(4), np.arange(4)) / 4) / 2.0
    rev = np.zeros((4, 4))
    rev[0, 0] = rev[3, 3] = rev[1, 2] = rev[2, 1] = 1
    assert np.abs(O.qft_dense(4, sites=[0, 1]) - np.kron(rev @ dft4, np.eye(4))).max() < 1e-12


@pytest.mark.parametrize("sites", [None, [0, 1], [1, 3, 4], [2]])
@pytest.mark.parametrize("inverse", [False, True])
def test_host_layers_match_oracle_circuit(sites, inverse):
    from paper_2601_16734_b200 import qft as Q
    L = 5
    ops = Q.qft_mpo(L, inverse, sites)
    subset = list(range(L)) if sites is None else sites
    assert ops.terms() == len(subset)
    U = np.eye(1 << L)
    for k in range(ops.terms() - 1, -1, -1):  # last factor acts first
        layer = ops[k]
        assert max(max(t.shape[0], t.shape[3]) for t in layer) <= 2
        U = O.mpo_to_dense(O.MPO(layer)) @ U
    assert np.abs(U - O.qft_dense(L, inverse, subset)).max() < 1e-13


def test_host_qft_errors_and_flip():
    from paper_2601_16734_b200 import qft as Q
    from paper_2601_16734_b200 import ttlab
    for bad in ([], [1, 1], [2, 1], [-1, 2], [0, 5]):
        with pytest.raises(ttlab.ShapeError):
            Q.qft_mpo(5, False, bad)
    with pytest.raises(ttlab.ShapeError):
        Q.qft_mpo(0)
    v = O.random_uniform_mps(5, 2, 3, 25)  # involution (test_lapack.cpp:313-316)
    assert np.array_equal(O.mps_to_dense(O.MPS(Q.qft_flip(Q.qft_flip(v.tensors)))), O.mps_to_dense(v))
    assert np.abs(O.mps_to_dense(O.MPS(Q.qft_flip(v.tensors))) - O.bit_reversal(5) @ O.mps_to_dense(v)).max() < 1e-13
