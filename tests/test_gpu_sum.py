"""§8f rows 1-2 on the GPU: MPSSum join, combine / simplify(MPSSum),
apply(MPO, MPSSum) and apply(MPOList, ...) against the oracle and the
reference's own cases (test_blas.cpp:8-36, 67-71, 132-141)."""
import numpy as np
import pytest

from oracle import ttlab_oracle as O
from oracle.rng import random_matrix
from paper_2601_16734_b200 import inputs as I

from ._compare import dense, distance, rel

pytestmark = pytest.mark.gpu


def T():
    from paper_2601_16734_b200 import ttlab
    return ttlab


def omps(tensors, err=0.0):
    return O.MPS([np.asarray(t) for t in tensors], err)


def _three_terms():
    states = [O.random_uniform_mps(5, 2, 2, 3), O.random_uniform_mps(5, 2, 3, 4), O.random_uniform_mps(5, 2, 2, 5)]
    w = [0.3 - 1.0j, -2.0 + 0.1j, 0.7j]
    return w, states


def test_join_is_exact_block_concatenation():
    """mps.hpp:352-405, element for element (the joined tensors are exact)."""
    t = T()
    w, states = _three_terms()
    got = t.MPSSum(w, [s.tensors for s in states]).join()
    ref = O.MPSSum(w, states).join()
    assert got.bond_dimensions() == ref.bond_dimensions()
    for x, y in zip(got.to_tensors(), ref.tensors):
        assert x.shape == y.shape
        assert np.abs(x - y).max() <= 1e-15 * max(np.abs(y).max(), 1e-300) * 4
    # real weights keep real tensors; error = sum |w| err (mps.hpp:344-349)
    a = I.random_mps(6, 2, 4, 1)
    b = I.random_mps(6, 2, 3, 2)
    da, db = t.DeviceMPS.from_tensors(a, error=1e-3), t.DeviceMPS.from_tensors(b, error=2e-3)
    j = t.MPSSum([2.0, -0.5], [da, db]).join()
    assert j.to_tensors()[0].dtype == np.float64
    assert abs(j.error() - (2.0 * 1e-3 + 0.5 * 2e-3)) < 1e-18
    ref = O.MPSSum([2.0, -0.5], [omps(a), omps(b)]).join()
    assert np.abs(dense(j.to_tensors()) - O.mps_to_dense(ref)).max() < 1e-13
    # single term = scaled (mps.hpp:98-117), zero weight = zero_like
    s1 = t.MPSSum([-3.0j], [a]).join()
    assert np.abs(dense(s1.to_tensors()) - (-3.0j) * dense(a)).max() < 1e-13
    z = t.MPSSum([0.0], [a]).join()
    assert z.bond_dimensions() == [1] * 7 and np.abs(dense(z.to_tensors())).max() == 0.0


def test_combine_reference_cases():
    """test_blas.cpp:8-36."""
    t = T()
    v = O.random_uniform_mps(4, 2, 2, 1)
    s = t.combine([1.0, 1.0], [v.tensors, v.tensors])
    assert np.abs(dense(s.to_tensors()) - 2.0 * O.mps_to_dense(v)).max() < 1e-12
    v = O.random_uniform_mps(4, 2, 2, 2)
    d = t.combine([1.0, -1.0], [v.tensors, v.tensors])
    assert t.norm(d)[0] <= 1e-12
    w, states = _three_terms()
    e = sum(wl * O.mps_to_dense(st) for wl, st in zip(w, states))
    s = t.combine(w, [x.tensors for x in states], t.DEFAULT_STRATEGY.with_max_sweeps(8))
    assert np.linalg.norm(dense(s.to_tensors()) - e) < 1e-10
    assert np.linalg.norm(dense(s.to_tensors()) - e) <= s.error()
    s = t.combine(w, [x.tensors for x in states], t.NO_TRUNCATION)
    assert np.linalg.norm(dense(s.to_tensors()) - e) < 1e-10
    with pytest.raises(t.ShapeError):
        t.combine([], [])
    with pytest.raises(t.ShapeError):
        t.combine([1.0], [O.random_uniform_mps(3, 2, 1, 1).tensors, O.random_uniform_mps(3, 2, 1, 2).tensors])
    with pytest.raises(t.ShapeError):
        t.combine([1.0, 1.0], [O.random_uniform_mps(3, 2, 1, 1).tensors, O.random_uniform_mps(3, 3, 1, 2).tensors])


def test_simplify_sum_v_minus_v():
    """test_blas.cpp:67-71."""
    t = T()
    v = O.random_uniform_mps(4, 2, 3, 9)
    s = t.simplify(t.MPSSum([1.0, -1.0], [v.tensors, v.tensors]))
    assert t.norm(s)[0] <= 1e-12
    assert s.bond_dimensions() == [1] * 5


@pytest.mark.parametrize("cplx", [False, True])
def test_simplify_sum_parity_truncated(cplx):
    """Bounded-rank combination: same residual, error ledger, sweeps and
    state (gauge-invariant distance) as the oracle's CompressionEngine with
    per-term environments (simplify.hpp:15-131, 198-215)."""
    t = T()
    L = 10
    terms = [I.random_mps(L, 2, 8, 11, complex_=cplx), I.random_mps(L, 2, 6, 12, complex_=cplx),
             I.random_mps(L, 2, 5, 13, complex_=cplx)]
    w = [1.0, -0.7, 0.4 + (0.3j if cplx else 0.0)]
    strat = t.DEFAULT_STRATEGY.with_max_bond(8).with_max_sweeps(6)
    rep = []
    got = t.simplify(t.MPSSum(w, terms), strat, report=rep)
    orep = {}
    ref = O.simplify_sum(O.MPSSum(w, [omps(x) for x in terms]), O.DEFAULT_STRATEGY.with_max_bond(8).with_max_sweeps(6),
                         report=orep)
    tn = np.sqrt(orep["target_norm2"])
    assert abs(rep[0]["target_norm2"] - orep["target_norm2"]) <= 1e-12 * orep["target_norm2"]
    hist = orep["dist2"]  # the plateau rule (simplify.hpp:123) may fire one sweep apart at round-off level
    assert rep[0]["sweeps"] == orep["sweeps"] or (
        abs(rep[0]["sweeps"] - orep["sweeps"]) == 1 and abs(hist[-1] - hist[-2]) <= 1e-12 * orep["target_norm2"])
    assert abs(rep[0]["residual"] - orep["residual"]) <= 1e-10 * tn
    assert abs(got.error() - ref.error) <= 1e-10 * max(ref.error, 1e-300) + 1e-12
    assert got.bond_dimensions() == ref.bond_dimensions()
    gt = got.to_tensors()
    assert distance(gt, ref.tensors) <= 1e-10 * tn
    # the residual is the true distance to the dense sum
    e = sum(wl * dense(x) for wl, x in zip(w, terms))
    assert abs(np.linalg.norm(dense(gt) - e) - rep[0]["residual"]) <= 1e-8 * tn


def test_simplify_sum_guess_and_single_site():
    t = T()
    w, states = _three_terms()
    e = sum(wl * O.mps_to_dense(st) for wl, st in zip(w, states))
    g = O.basis_state(5, 2, 0)
    s = t.simplify(t.MPSSum(w, [x.tensors for x in states]), t.DEFAULT_STRATEGY.with_max_sweeps(8), guess=g.tensors)
    assert np.linalg.norm(dense(s.to_tensors()) - e) < 1e-9 * np.linalg.norm(e)
    # one-site chains: the terms are added (simplify.hpp:62-70)
    a, b = O.random_uniform_mps(1, 3, 1, 1), O.random_uniform_mps(1, 3, 1, 2)
    s = t.simplify(t.MPSSum([2.0, 1.0j], [a.tensors, b.tensors]), t.DEFAULT_STRATEGY.with_normalize(False))
    assert np.abs(dense(s.to_tensors()) - (2.0 * O.mps_to_dense(a) + 1.0j * O.mps_to_dense(b))).max() < 1e-14
    with pytest.raises(t.ShapeError):  # join of one-site chains (mps.hpp:129-133)
        t.MPSSum([1.0, 1.0], [a.tensors, b.tensors]).join()


def test_apply_mpo_to_sum():
    """blas.hpp:13-20 against the dense oracle and the oracle's apply_sum."""
    t = T()
    v1, v2 = O.random_uniform_mps(6, 2, 3, 12), O.random_uniform_mps(6, 2, 2, 17)
    a = O.mpo_sum([1 + 0.5j, -0.3], [O.mpo_from_local_operators([random_matrix(2, 2, s) for s in range(21, 27)]),
                                     O.mpo_identity(6, 2)])
    w = [0.5, 1.0 - 1.0j]
    e = O.mpo_to_dense(a) @ (w[0] * O.mps_to_dense(v1) + w[1] * O.mps_to_dense(v2))
    s = t.apply(a.tensors, t.MPSSum(w, [v1.tensors, v2.tensors]), t.DEFAULT_STRATEGY.with_max_sweeps(8))
    assert np.linalg.norm(dense(s.to_tensors()) - e) < 1e-10 * np.linalg.norm(e)
    ref = O.apply_sum(a, O.MPSSum(w, [v1, v2]), O.DEFAULT_STRATEGY.with_max_sweeps(8))
    # exact representation: residual = sqrt(max(0, <T,T> - |psi|^2)) is rounding
    # noise of size ~sqrt(eps)|T| on both sides (simplify.hpp:90, 126)
    assert abs(s.error() - ref.error) <= 1e-7 * np.linalg.norm(e)
    assert np.linalg.norm(dense(s.to_tensors()) - e) <= s.error() + 1e-12


def test_apply_mpolist_order():
    """test_blas.cpp:132-141 plus a bounded-bond chain of Laplacians against the oracle."""
    t = T()
    v = O.random_uniform_mps(3, 2, 2, 13)
    m1, m2 = random_matrix(2, 2, 31), random_matrix(2, 2, 32)
    i2 = np.eye(2)
    a = O.mpo_from_local_operators([m1, i2, i2])
    b = O.mpo_from_local_operators([m2, i2, i2])
    e = O.mpo_to_dense(a) @ (O.mpo_to_dense(b) @ O.mps_to_dense(v))
    out = t.apply(t.MPOList([a.tensors, b.tensors]), v.tensors)
    assert np.linalg.norm(dense(out.to_tensors()) - e) < 1e-10
    with pytest.raises(t.ShapeError):
        t.apply(t.MPOList([]), v.tensors)
    psi = I.random_mps(10, 2, 8, 5)
    W = I.laplacian_mpo(10)
    strat = t.DEFAULT_STRATEGY.with_max_bond(8).with_max_sweeps(4)
    got = t.apply(t.MPOList([W, W, W]), psi, strat)
    ref = O.apply_list([O.MPO(W)] * 3, omps(psi), O.DEFAULT_STRATEGY.with_max_bond(8).with_max_sweeps(4))
    assert got.bond_dimensions() == ref.bond_dimensions()
    tn = ref.norm()
    assert distance(got.to_tensors(), ref.tensors) <= 1e-9 * max(tn, 1.0)
    assert abs(got.error() - ref.error) <= 1e-9 * max(ref.error, 1.0)
