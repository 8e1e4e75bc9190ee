"""Pins the CPU oracle against the reference's own known-answer tests for the
hot path (re-expressed from /root/reference/proj/tests/*.cpp, same tolerances)
and its input generator against golden vectors from libstdc++."""
import json
import os
import struct

import numpy as np
import pytest

from oracle import ttlab_oracle as O
from oracle.rng import MT19937_64, complex_draws, random_matrix

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _hexd(s):
    return struct.unpack("<d", bytes.fromhex(s)[::-1])[0]


def test_mt19937_64_matches_libstdcxx():
    g = json.load(open(os.path.join(GOLDEN, "mt19937_64_uniform.json")))
    for seed, v in g.items():
        raw = MT19937_64(int(seed)).draw(8)
        assert [f"{int(x):016x}" for x in raw] == v["raw"]
        z = complex_draws(MT19937_64(int(seed)), len(v["cplx"]))
        exp = np.array([_hexd(a) + 1j * _hexd(b) for a, b in v["cplx"]])
        assert np.array_equal(z, exp)


def test_random_uniform_mps_shapes():
    """test_core.cpp random_uniform_mps section."""
    assert O.random_uniform_mps(3, 2, 1, 5).max_bond_dimension() == 1
    a, b = O.random_uniform_mps(4, 2, 3, 99), O.random_uniform_mps(4, 2, 3, 99)
    assert all(np.array_equal(x, y) for x, y in zip(a.tensors, b.tensors))
    assert O.random_uniform_mps(4, 2, 16, 1).bond_dimensions() == [1, 2, 4, 2, 1]


def test_schmidt_split_kats():
    """test_core.cpp:73-101."""
    th = np.eye(2) / np.sqrt(2)
    a, b, err = O.schmidt_split(th, O.NO_TRUNCATION)
    assert err == 0.0
    assert np.linalg.norm(a @ b - th) < 1e-14
    s = O.schmidt_values(th)
    assert abs(s[0] - 1 / np.sqrt(2)) < 1e-15 and abs(s[1] - 1 / np.sqrt(2)) < 1e-15
    a, b, err = O.schmidt_split(th, O.NO_TRUNCATION.with_max_bond(1))
    assert abs(err - 1 / np.sqrt(2)) < 1e-15 and a.shape[1] == 1
    th = random_matrix(4, 4, 5)
    a, b, err = O.schmidt_split(th, O.NO_TRUNCATION.with_max_bond(2))
    assert abs(np.linalg.norm(a @ b - th) - err) < 1e-12
    th = random_matrix(6, 4, 9)
    a, b, _ = O.schmidt_split(th, O.NO_TRUNCATION, O.LEFT_TO_RIGHT)
    assert np.linalg.norm(a.conj().T @ a - np.eye(4)) < 1e-12
    a, b, _ = O.schmidt_split(th, O.NO_TRUNCATION, O.RIGHT_TO_LEFT)
    assert np.linalg.norm(b @ b.conj().T - np.eye(4)) < 1e-12


def _check_iso(c):
    for n, A in enumerate(c.tensors):
        if n < c.center:
            a = A.reshape(-1, A.shape[2])
            assert np.linalg.norm(a.conj().T @ a - np.eye(a.shape[1])) <= 1e-12
        elif n > c.center:
            b = A.reshape(A.shape[0], -1)
            assert np.linalg.norm(b @ b.conj().T - np.eye(b.shape[0])) <= 1e-12


def test_canonicalize_pins():
    """test_core.cpp:119-155."""
    state = O.random_uniform_mps(6, 2, 5, 42)
    for center in (0, 2, 5):
        c = O.canonicalize(state, center, O.NO_TRUNCATION)
        assert c.center == center
        _check_iso(c)
        assert np.abs(O.mps_to_dense(c) - O.mps_to_dense(state)).max() < 1e-12
    state = O.random_uniform_mps(8, 2, 8, 3)
    exact = O.mps_to_dense(state)
    c = O.canonicalize(state, 3, O.NO_TRUNCATION.with_max_bond(4))
    dist = np.linalg.norm(O.mps_to_dense(c) - exact)
    assert dist <= c.error
    assert abs(dist - c.error) < 1e-10 * np.linalg.norm(exact)
    assert c.max_bond_dimension() <= 4
    _check_iso(c)
    state = O.random_uniform_mps(6, 2, 4, 11)
    exact = O.mps_to_dense(state)
    c = O.canonicalize(state, 0, O.NO_TRUNCATION)
    c.recenter(5, O.NO_TRUNCATION)
    c.recenter(0, O.NO_TRUNCATION)
    assert np.linalg.norm(O.mps_to_dense(c) - exact) < 1e-12 * np.linalg.norm(exact)


def test_norms():
    """test_core.cpp:157-174."""
    assert abs(O.basis_state(5, 2, 0).norm() - 1) < 1e-15
    s = O.random_uniform_mps(5, 2, 3, 17)
    assert abs(s.scaled(2.0).norm() - 2 * s.norm()) < 1e-12 * s.norm()
    assert abs(s.scaled(-3j).norm() - 3 * s.norm()) < 1e-12 * s.norm()
    s = O.random_uniform_mps(6, 2, 4, 23)
    assert abs(s.norm() - np.linalg.norm(O.mps_to_dense(s))) < 1e-12 * s.norm()
    assert abs(O.canonicalize(s, 2, O.NO_TRUNCATION).norm() - s.norm()) < 1e-12 * s.norm()


def test_apply_raw_pins():
    """test_core.cpp:200-227."""
    s = O.random_uniform_mps(5, 2, 3, 21)
    assert np.abs(O.mps_to_dense(O.apply_raw(O.mpo_identity(5, 2), s)) - O.mps_to_dense(s)).max() < 1e-14
    st = O.random_uniform_mps(4, 2, 3, 31)
    a = O.mpo_from_local_operators([random_matrix(2, 2, k) for k in (1, 2, 3, 4)])
    b = O.mpo_from_local_operators([random_matrix(2, 2, k) for k in (5, 6, 7, 8)])
    m = O.mpo_sum([0.5 + 0.25j, -1 + 1j], [a, b])
    assert np.abs(O.mps_to_dense(O.apply_raw(m, st)) - O.mpo_to_dense(m) @ O.mps_to_dense(st)).max() < 1e-12


def test_error_ledger():
    """test_core.cpp:258-265."""
    state = O.random_uniform_mps(6, 2, 6, 55)
    c1 = O.canonicalize(state, 0, O.NO_TRUNCATION.with_max_bond(3))
    c2 = O.canonicalize(O.MPS(c1.tensors, c1.error), 0, O.NO_TRUNCATION.with_max_bond(2))
    assert c2.error >= c1.error
    assert np.linalg.norm(O.mps_to_dense(c2) - O.mps_to_dense(state)) <= c2.error


def test_simplify_pins():
    """test_blas.cpp:40-77."""
    v = O.random_uniform_mps(6, 2, 4, 7)
    s = O.simplify(v, O.DEFAULT_STRATEGY.with_max_sweeps(6))
    assert np.linalg.norm(O.mps_to_dense(s) - O.mps_to_dense(v)) < 1e-10 * v.norm()
    v = O.random_uniform_mps(6, 2, 8, 8)
    d = O.mps_to_dense(v)
    s = O.simplify(v, O.DEFAULT_STRATEGY.with_max_bond(4).with_max_sweeps(12))
    assert s.max_bond_dimension() <= 4
    dist = np.linalg.norm(O.mps_to_dense(s) - d)
    sv = np.linalg.svd(d.reshape(8, 8), compute_uv=False)
    lower = np.sqrt(np.sum(sv[4:] ** 2))
    assert lower - 1e-12 <= dist <= 1.10 * max(lower, 1e-14)
    assert abs(s.error - dist) < 1e-8 * np.linalg.norm(d)
    v = O.random_uniform_mps(5, 2, 3, 10)
    s = O.simplify(v, O.DEFAULT_STRATEGY.with_max_sweeps(8), O.basis_state(5, 2, 0))
    assert np.linalg.norm(O.mps_to_dense(s) - O.mps_to_dense(v)) < 1e-9 * v.norm()
    v = O.random_uniform_mps(4, 2, 3, 9)  # combine v - v -> 0 (test_blas.cpp:68-71 via MPSSum)
    assert O.combine([1.0, -1.0], [v, v]).norm() <= 1e-12


def test_combine_pins():
    """test_blas.cpp:8-36 (combine), 67-71 (simplify(MPSSum)), 132-141 (MPOList)."""
    v = O.random_uniform_mps(4, 2, 2, 1)
    s = O.combine([1.0, 1.0], [v, v])
    assert np.abs(O.mps_to_dense(s) - 2.0 * O.mps_to_dense(v)).max() < 1e-12
    v = O.random_uniform_mps(4, 2, 2, 2)
    assert O.combine([1.0, -1.0], [v, v]).norm() <= 1e-12
    states = [O.random_uniform_mps(5, 2, 2, 3), O.random_uniform_mps(5, 2, 3, 4), O.random_uniform_mps(5, 2, 2, 5)]
    w = [0.3 - 1.0j, -2.0 + 0.1j, 0.7j]
    e = sum(wl * O.mps_to_dense(st) for wl, st in zip(w, states))
    s = O.combine(w, states, O.DEFAULT_STRATEGY.with_max_sweeps(8))
    assert np.linalg.norm(O.mps_to_dense(s) - e) < 1e-10
    assert np.linalg.norm(O.mps_to_dense(s) - e) <= s.error
    s = O.combine(w, states, O.NO_TRUNCATION)
    assert np.linalg.norm(O.mps_to_dense(s) - e) < 1e-10
    with pytest.raises(O.ShapeError):
        O.combine([], [])
    with pytest.raises(O.ShapeError):
        O.combine([1.0], [O.random_uniform_mps(3, 2, 1, 1), O.random_uniform_mps(3, 2, 1, 2)])
    v = O.random_uniform_mps(4, 2, 3, 9)
    assert O.simplify_sum(O.MPSSum([1.0, -1.0], [v, v])).norm() <= 1e-12
    # join is the exact block concatenation (mps.hpp:352-405)
    j = O.MPSSum(w, states).join()
    assert np.abs(O.mps_to_dense(j) - e).max() < 1e-12
    bsum = [sum(x) for x in zip(*[st.bond_dimensions() for st in states])]
    assert j.bond_dimensions() == [1] + bsum[1:-1] + [1]
    v = O.random_uniform_mps(3, 2, 2, 13)
    m1, m2 = random_matrix(2, 2, 31), random_matrix(2, 2, 32)
    i2 = np.eye(2)
    a = O.mpo_from_local_operators([m1, i2, i2])
    b = O.mpo_from_local_operators([m2, i2, i2])
    e = O.mpo_to_dense(a) @ (O.mpo_to_dense(b) @ O.mps_to_dense(v))
    assert np.linalg.norm(O.mps_to_dense(O.apply_list([a, b], v)) - e) < 1e-10


def test_apply_and_hadamard_pins():
    """test_blas.cpp:108-142, 181-202."""
    v = O.random_uniform_mps(5, 2, 3, 11)
    w = O.apply(O.mpo_identity(5, 2), v)
    assert np.linalg.norm(O.mps_to_dense(w) - O.mps_to_dense(v)) <= 1e-12 * v.norm()
    v = O.random_uniform_mps(6, 2, 3, 12)
    a = O.mpo_sum([1 + 0.5j, -0.3], [O.mpo_from_local_operators([random_matrix(2, 2, s) for s in range(21, 27)]),
                                     O.mpo_identity(6, 2)])
    e = O.mpo_to_dense(a) @ O.mps_to_dense(v)
    w = O.apply(a, v, O.DEFAULT_STRATEGY.with_max_sweeps(8))
    assert np.linalg.norm(O.mps_to_dense(w) - e) < 1e-10 * np.linalg.norm(e)
    with pytest.raises(O.ShapeError):
        O.apply(O.mpo_identity(3, 2), O.random_uniform_mps(4, 2, 1, 1))
    with pytest.raises(O.ShapeError):
        O.apply(O.mpo_identity(4, 3), O.random_uniform_mps(4, 2, 1, 1))
    u, v = O.random_uniform_mps(5, 2, 2, 20), O.random_uniform_mps(5, 2, 3, 21)
    w = O.hadamard(u, v)
    assert np.abs(O.mps_to_dense(w) - O.mps_to_dense(u) * O.mps_to_dense(v)).max() < 1e-12
    assert w.bond_dimensions() == [x * y for x, y in zip(u.bond_dimensions(), v.bond_dimensions())]
    e1, e2 = O.basis_state(3, 2, 1), O.basis_state(3, 2, 2)
    assert np.linalg.norm(O.mps_to_dense(O.hadamard(e1, e2))) == 0.0


def test_two_site_linear_form_pins_projection():
    """test_blas.cpp:289-299: <v, w> from the projected pair at any site, both
    contraction orders of project_pair (forms.hpp:13-32)."""
    v = O.random_uniform_mps(6, 2, 3, 30)
    w = O.random_uniform_mps(6, 2, 2, 31)
    ref = O.scprod(v, w)
    for n in (0, 2, 4):
        L = np.ones((1, 1), dtype=complex)
        for k in range(n):
            L = O.update_left_environment(L, v[k], w[k])
        R = np.ones((1, 1), dtype=complex)
        for k in range(5, n + 1, -1):
            R = O.update_right_environment(R, v[k], w[k])
        for proj in (O.project_pair, O.project_pair_fast):
            f = proj(L, w[n], w[n + 1], R)
            pair = O.join_pair(v[n], v[n + 1])
            assert abs(np.vdot(pair, f) - ref) < 1e-12


def test_expectation_pins():
    """test_blas.cpp:155-178 against dense contractions."""
    sz = np.diag([1.0, -1.0])
    assert abs(O.expectation_local(O.basis_state(3, 2, 0), sz, 0) - 1.0) < 1e-15
    assert abs(O.expectation_local(O.basis_state(2, 2, 1), sz, 0, sz, 1) + 1.0) < 1e-15
    v = O.random_uniform_mps(4, 2, 3, 16)
    d = O.mps_to_dense(v)
    op, op2 = random_matrix(2, 2, 40), random_matrix(2, 2, 41)
    emb = lambda m, k: np.kron(np.kron(np.eye(2 ** k), m), np.eye(2 ** (3 - k)))
    assert abs(O.expectation_local(v, op, 2) - np.vdot(d, emb(op, 2) @ d)) < 1e-12
    assert abs(O.expectation_local(v, op, 1, op2, 3) - np.vdot(d, emb(op, 1) @ emb(op2, 3) @ d)) < 1e-12
    u, w = O.random_uniform_mps(4, 2, 2, 17), O.random_uniform_mps(4, 2, 3, 18)
    assert abs(O.expectation_mpo(O.mpo_identity(4, 2), u, w) - O.scprod(u, w)) < 1e-12
    mpo = O.mpo_from_local_operators([random_matrix(2, 2, s) for s in (51, 52, 53, 54)])
    ref = np.vdot(O.mps_to_dense(u), O.mpo_to_dense(mpo) @ O.mps_to_dense(w))
    assert abs(O.expectation_mpo(mpo, u, w) - ref) < 1e-12
    with pytest.raises(O.ShapeError):
        O.expectation_local(v, op, 4)
    with pytest.raises(O.ShapeError):
        O.expectation_local(v, op, 1, op2, 1)
    with pytest.raises(O.ShapeError):
        O.expectation_local(v, np.eye(3), 1)


def test_ttlab1_container_pins():
    """test_core.cpp:229-256 (bit-exact round trip, bad magic) and the byte layout
    of serialize.hpp:13-16 assembled independently with struct."""
    import struct
    state = O.random_uniform_mps(5, 2, 4, 123)
    state.error = 0.125
    blob = O.dumps_mps(state)
    back = O.loads_mps(blob)
    assert back.error == 0.125 and len(back) == 5
    for a, b in zip(back.tensors, state.tensors):
        assert a.shape == b.shape and a.tobytes() == b.astype(np.complex128).tobytes()
    t0 = state.tensors[0]
    head = b"TTLAB1\0" + struct.pack("<I", 1) + struct.pack("<I", 5)
    rec0 = struct.pack("<B", 3) + struct.pack("<QQQ", *t0.shape)
    assert blob.startswith(head + rec0)
    assert blob[len(head) + len(rec0):len(head) + len(rec0) + 16] == struct.pack("<dd", t0[0, 0, 0].real, t0[0, 0, 0].imag)
    assert blob.endswith(struct.pack("<d", 0.125))
    op = O.mpo_identity(3, 2)
    ob = O.loads_mpo(O.dumps_mpo(op))
    assert all(np.array_equal(a, b) for a, b in zip(ob.tensors, op.tensors))
    with pytest.raises(O.NumericError):
        O.loads_mps(b"garbage")
    with pytest.raises(O.NumericError):
        O.loads_mps(blob[:-9])
    with pytest.raises(O.NumericError):
        O.loads_mps(O.dumps_mpo(op))  # rank-4 record in an MPS file
