"""CanonicalMPS centre moves and schmidt_split on the device against the oracle
(mps.hpp:238-279, 316-323; schmidt.hpp:72-89)."""
import numpy as np
import pytest

from oracle import ttlab_oracle as O

from ._compare import dense, rel

pytestmark = pytest.mark.gpu


def T():
    from paper_2601_16734_b200 import ttlab
    return ttlab


def _isometries(tensors, center):
    for n, A in enumerate(tensors):
        if n < center:
            a = A.reshape(-1, A.shape[2])
            assert np.abs(a.conj().T @ a - np.eye(a.shape[1])).max() <= 1e-12
        elif n > center:
            b = A.reshape(A.shape[0], -1)
            assert np.abs(b @ b.conj().T - np.eye(b.shape[0])).max() <= 1e-12


@pytest.mark.parametrize("complex_", [False, True])
@pytest.mark.parametrize("direction", [0, 1])
def test_schmidt_split_matches_oracle(complex_, direction):
    t = T()
    rng = np.random.default_rng(3 + direction)
    for (m, n, mb) in [(6, 4, None), (40, 64, 10), (300, 200, 50), (2, 2, 1)]:
        th = rng.standard_normal((m, n))
        if complex_:
            th = th + 1j * rng.standard_normal((m, n))
        strat = t.Strategy(max_bond=mb) if mb else t.NO_TRUNCATION
        ostrat = O.Strategy(max_bond=mb) if mb else O.NO_TRUNCATION
        a, b, err = t.schmidt_split(th, strat, direction)
        ra, rb, rerr = O.schmidt_split(th, ostrat, direction)
        assert a.shape == ra.shape and b.shape == rb.shape
        assert abs(err - rerr) <= 1e-12 * np.linalg.norm(th)
        assert np.abs(a @ b - ra @ rb).max() <= 1e-12 * np.linalg.norm(th)
        if direction == 0:
            assert np.abs(a.conj().T @ a - np.eye(a.shape[1])).max() < 1e-12
        else:
            assert np.abs(b @ b.conj().T - np.eye(b.shape[0])).max() < 1e-12


def test_recenter_exact_and_truncating():
    """test_core.cpp:148-155 (exact moves) and truncating moves against the oracle's recenter."""
    t = T()
    state = O.random_uniform_mps(6, 2, 4, 11)
    exact = O.mps_to_dense(state)
    c = t.canonicalize(state.tensors, 0, t.NO_TRUNCATION)
    c5, err = t.recenter(c, 5, t.NO_TRUNCATION)
    assert c5.center == 5 and err < 1e-12
    _isometries(c5.to_tensors(), 5)
    c0, _ = t.recenter(c5, 0, t.NO_TRUNCATION)
    assert rel(dense(c0.to_tensors()), exact) < 1e-12
    # truncating moves (max_bond 3) from centre 0 to 7
    state = O.random_uniform_mps(8, 2, 8, 3)
    c = t.canonicalize(state.tensors, 0, t.NO_TRUNCATION)
    moved, err = t.recenter(c, 7, t.NO_TRUNCATION.with_max_bond(3))
    ref = O.canonicalize(state, 0, O.NO_TRUNCATION)
    ref_err0 = ref.error
    ref.recenter(7, O.NO_TRUNCATION.with_max_bond(3))
    assert moved.bond_dimensions() == ref.bond_dimensions()
    assert abs(err - (ref.error - ref_err0)) <= 1e-12
    _isometries(moved.to_tensors(), 7)
    assert rel(dense(moved.to_tensors()), O.mps_to_dense(ref)) <= 1e-10
    with pytest.raises(t.ShapeError):
        t.recenter(c, 8, t.NO_TRUNCATION)


def test_mps_from_device_validates_and_copies():
    """ttg_mps_from_device: device buffers (torch tensors on another stream) are copied before
    the call returns; bad dtype / shapes / errors are rejected."""
    import torch
    t = T()
    from paper_2601_16734_b200 import _lib
    psi = [np.random.default_rng(k).standard_normal(s) for k, s in enumerate([(1, 2, 3), (3, 2, 4), (4, 2, 1)])]
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        dev = [torch.from_numpy(a.copy()).cuda(non_blocking=True) for a in psi]
    bonds, phys = [1, 3, 4, 1], [2, 2, 2]
    m = t.DeviceMPS.from_device(3, _lib.TTG_F64, 1, bonds, phys, [d.data_ptr() for d in dev], [0.5])
    for d in dev:
        d.fill_(float("nan"))  # the copy is complete: overwriting the sources must not matter
    torch.cuda.synchronize()
    got = m.to_tensors()
    for a, b in zip(got, psi):
        assert np.array_equal(a, b)
    assert m.error() == 0.5
    ptrs = [d.data_ptr() for d in dev]
    with pytest.raises(Exception):
        t.DeviceMPS.from_device(3, 7, 1, bonds, phys, ptrs)  # unknown dtype
    with pytest.raises(t.ShapeError):
        t.DeviceMPS.from_device(3, _lib.TTG_F64, 1, [1, 0, 4, 1], phys, ptrs)
    with pytest.raises(t.ShapeError):
        t.DeviceMPS.from_device(3, _lib.TTG_F64, 1, bonds, phys, ptrs, [-1.0])
    with pytest.raises(t.ShapeError):  # scprod of states with different physical dimensions
        u = t.DeviceMPS.from_tensors([np.ones((1, 2, 1)), np.ones((1, 3, 1))])
        v = t.DeviceMPS.from_tensors([np.ones((1, 2, 1)), np.ones((1, 2, 1))])
        t.scprod(u, v)
