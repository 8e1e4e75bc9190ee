"""numpy/scipy restatement of the ttlab apply/hadamard + simplify hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Every function cites the
reference file:line it restates; paths are relative to
/root/reference/proj/include/ttlab/.

Dense linear algebra: the reference calls Eigen3 (unpinned "≥ 3.3",
proj/CMakeLists.txt:10; not vendored).  Eigen's `HouseholderQR` is restated with
LAPACK geqrf/orgqr (numpy.linalg.qr, reduced) and `JacobiSVD` (thin U, V) with
LAPACK gesvd (scipy, gesdd fallback).  All are backward stable, so every
gauge-invariant quantity agrees to O(eps * cond) with the reference.

Arithmetic: the reference is complex128 everywhere (types.hpp:12-16).  Tensors
here keep the dtype they are given; `promote=True` on the entry points casts
to complex128 first ("reference arithmetic", used for the timed CPU baseline).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import List, Optional, Sequence

import numpy as np
import scipy.linalg

EPS = np.finfo(np.float64).eps
UNBOUNDED_BOND = (1 << 63) - 1  # types.hpp:19
DENSE_VECTOR_GUARD = 1 << 26  # mps.hpp:15
DENSE_OPERATOR_GUARD = 1 << 13  # mpo.hpp:10

SVD_TRUNCATE, VARIATIONAL = 0, 1  # types.hpp:39

# Diagnostics: when a list, every truncating schmidt_split
# appends (rows, cols, rank, s_r-1, s_r, relative gap (s_{r-1} - s_r) / s_{r-1})
# for splits that drop singular values.  The gap decides how sensitive the kept
# subspace is to rounding, i.e. whether 1e-10 parity is reachable.
GAP_LOG: Optional[list] = None
LEFT_TO_RIGHT, RIGHT_TO_LEFT = 0, 1  # types.hpp:41


class ShapeError(ValueError):
    """types.hpp:22-25 shape_error."""


class CapacityError(RuntimeError):
    """types.hpp:28-31 capacity_error."""


class NumericError(RuntimeError):
    """types.hpp:34-37 numeric_error."""


@dataclass(frozen=True)
class Strategy:
    """types.hpp:50-88."""

    method: int = VARIATIONAL
    tolerance: float = 1e-12
    simplification_tolerance: float = 1e-12
    max_bond: int = UNBOUNDED_BOND
    max_sweeps: int = 4
    normalize: bool = False

    def with_method(self, m):
        return replace(self, method=m)

    def with_tolerance(self, t):
        return replace(self, tolerance=t)

    def with_simplification_tolerance(self, t):
        return replace(self, simplification_tolerance=t)

    def with_max_bond(self, chi):
        return replace(self, max_bond=chi)

    def with_max_sweeps(self, s):
        return replace(self, max_sweeps=s)

    def with_normalize(self, f):
        return replace(self, normalize=f)


DEFAULT_STRATEGY = Strategy()  # types.hpp:90
NO_TRUNCATION = Strategy(SVD_TRUNCATE, 0.0, 0.0, UNBOUNDED_BOND, 4, False)  # types.hpp:93-94


def fp_error_floor(scale: float) -> float:
    """types.hpp:100-102."""
    return 32.0 * EPS * scale


# ----------------------------------------------------------------------------
# containers (tensor.hpp:13-149, mps.hpp:21-143, mpo.hpp:14-105)
# ----------------------------------------------------------------------------


class MPS:
    """mps.hpp:21-143.  tensors[n] has shape (left, phys, right), row-major."""

    def __init__(self, tensors: Sequence[np.ndarray], error: float = 0.0):
        self.tensors = [np.asarray(t) for t in tensors]
        self.error = float(error)
        self._check_shape()

    def _check_shape(self):  # mps.hpp:129-139
        if not self.tensors:
            return
        if self.tensors[0].shape[0] != 1 or self.tensors[-1].shape[2] != 1:
            raise ShapeError("MPS boundary bonds must have size one")
        for a, b in zip(self.tensors[:-1], self.tensors[1:]):
            if a.shape[2] != b.shape[0]:
                raise ShapeError("MPS bond mismatch between neighboring tensors")
        if self.error < 0:
            raise ShapeError("MPS error bound must be non-negative")

    def __len__(self):
        return len(self.tensors)

    def __getitem__(self, n):
        return self.tensors[n]

    def copy(self):
        return type(self)([t.copy() for t in self.tensors], self.error)

    def bond_dimensions(self) -> List[int]:  # mps.hpp:45-52
        return [self.tensors[0].shape[0]] + [t.shape[2] for t in self.tensors]

    def physical_dimensions(self) -> List[int]:
        return [t.shape[1] for t in self.tensors]

    def max_bond_dimension(self) -> int:  # mps.hpp:54-59
        return max([1] + [max(t.shape[0], t.shape[2]) for t in self.tensors])

    def dimension(self, guard=DENSE_VECTOR_GUARD) -> int:  # mps.hpp:62-70
        dim = 1
        for t in self.tensors:
            dim *= t.shape[1]
            if dim > guard:
                raise CapacityError("MPS dimension exceeds guard")
        return dim

    def norm_squared(self) -> float:  # mps.hpp:80-85
        env = np.ones((1, 1), dtype=self.tensors[0].dtype)
        for t in self.tensors:
            env = update_left_environment(env, t, t)
        return float(np.real(env[0, 0]))

    def norm(self) -> float:  # mps.hpp:86
        return math.sqrt(max(0.0, self.norm_squared()))

    def scaled(self, factor) -> "MPS":  # mps.hpp:98-117
        L = len(self)
        mag = abs(factor)
        if mag == 0.0:
            return self.zero_like()
        root = mag ** (1.0 / L)
        phase = factor / mag
        out = []
        for n, t in enumerate(self.tensors):
            f = root * (phase if n == 0 else 1.0)
            if np.iscomplexobj(f) and not np.iscomplexobj(t):
                if f.imag == 0:
                    f = f.real
                else:
                    t = t.astype(np.complex128)
            out.append(t * f)
        return MPS(out, self.error * mag)

    def zero_like(self) -> "MPS":  # mps.hpp:120-126
        return MPS([np.zeros((1, t.shape[1], 1), dtype=t.dtype) for t in self.tensors], 0.0)


class CanonicalMPS(MPS):
    """mps.hpp:180-307."""

    def __init__(self, state: MPS, center: int, strategy: Strategy, _raw=False):
        super().__init__([t.copy() for t in state.tensors], state.error)
        self.center = 0
        if _raw:
            self.center = center
            return
        L = len(self)
        if center < 0 or center >= L:
            raise ShapeError("canonical center out of range")
        T = self.tensors
        # Pass 1: exact left-to-right QR (mps.hpp:193-205)
        for n in range(L - 1):
            a, d, b = T[n].shape
            q, r = np.linalg.qr(T[n].reshape(a * d, b), mode="reduced")
            rank = min(a * d, b)
            nxt = T[n + 1]
            carried = r @ nxt.reshape(nxt.shape[0], -1)
            T[n + 1] = carried.reshape(rank, nxt.shape[1], nxt.shape[2])
            T[n] = q.reshape(a, d, rank)
        # Pass 2: truncating right-to-left (mps.hpp:206-210)
        err2 = 0.0
        self.center = L - 1
        while self.center > 0:
            err2 += self.move_center_left(strategy) ** 2
        # Pass 3 (mps.hpp:211-213)
        while self.center < center:
            err2 += self.move_center_right(strategy) ** 2
        self.error += math.sqrt(err2) + fp_error_floor(self.norm())  # mps.hpp:214-215
        if strategy.normalize:
            self.normalize_in_place()

    @classmethod
    def raw(cls, tensors, center, error=0.0):
        return cls(MPS(tensors, error), center, NO_TRUNCATION, _raw=True)

    def norm_squared(self) -> float:  # mps.hpp:222-224
        return float(np.vdot(self.tensors[self.center], self.tensors[self.center]).real)

    def norm(self) -> float:  # mps.hpp:225
        return float(np.linalg.norm(self.tensors[self.center]))

    def normalize_in_place(self):  # mps.hpp:227-235
        n = self.norm()
        if n == 0.0:
            return
        self.tensors[self.center] = self.tensors[self.center] / n
        self.error /= n

    def move_center_right(self, strategy) -> float:  # mps.hpp:238-250
        c = self.center
        if c + 1 >= len(self):
            raise ShapeError("move_center_right: already at the last site")
        t = self.tensors[c]
        a_, d_, b_ = t.shape
        a, b, err = schmidt_split(t.reshape(a_ * d_, b_), strategy, LEFT_TO_RIGHT)
        rank = a.shape[1]
        self.tensors[c] = a.reshape(a_, d_, rank)
        nxt = self.tensors[c + 1]
        carried = b @ nxt.reshape(nxt.shape[0], -1)
        self.tensors[c + 1] = carried.reshape(rank, nxt.shape[1], nxt.shape[2])
        self.center += 1
        return err

    def move_center_left(self, strategy) -> float:  # mps.hpp:253-265
        c = self.center
        if c == 0:
            raise ShapeError("move_center_left: already at the first site")
        t = self.tensors[c]
        a_, d_, b_ = t.shape
        a, b, err = schmidt_split(t.reshape(a_, d_ * b_), strategy, RIGHT_TO_LEFT)
        rank = b.shape[0]
        self.tensors[c] = b.reshape(rank, d_, b_)
        prev = self.tensors[c - 1]
        carried = prev.reshape(-1, prev.shape[2]) @ a
        self.tensors[c - 1] = carried.reshape(prev.shape[0], prev.shape[1], rank)
        self.center -= 1
        return err

    def recenter(self, target, strategy):  # mps.hpp:268-279
        if target < 0 or target >= len(self):
            raise ShapeError("recenter: center out of range")
        err2 = 0.0
        while self.center < target:
            err2 += self.move_center_right(strategy) ** 2
        while self.center > target:
            err2 += self.move_center_left(strategy) ** 2
        if err2 > 0:
            self.error += math.sqrt(err2)
        return self

    def update_two_site(self, joined, direction, strategy) -> float:  # mps.hpp:283-297
        n = self.center
        to_right = direction == LEFT_TO_RIGHT
        if (to_right and n + 1 >= len(self)) or ((not to_right) and n == 0):
            raise ShapeError("update_two_site: no neighboring pair in that direction")
        lo = n if to_right else n - 1
        d1 = self.tensors[lo].shape[1]
        d2 = self.tensors[lo + 1].shape[1]
        left, right, err = split_pair(joined, d1, d2, strategy, direction)
        self.tensors[lo] = left
        self.tensors[lo + 1] = right
        self.center = lo + 1 if to_right else lo
        return err


def canonicalize(state: MPS, center: int = 0, strategy: Strategy = DEFAULT_STRATEGY) -> CanonicalMPS:
    """mps.hpp:310-313."""
    return CanonicalMPS(state, center, strategy)


class MPO:
    """mpo.hpp:14-105.  tensors[n] has shape (left, out, in, right)."""

    def __init__(self, tensors: Sequence[np.ndarray]):
        self.tensors = [np.asarray(t) for t in tensors]
        if self.tensors:
            if self.tensors[0].shape[0] != 1 or self.tensors[-1].shape[3] != 1:
                raise ShapeError("MPO boundary bonds must have size one")
            for a, b in zip(self.tensors[:-1], self.tensors[1:]):
                if a.shape[3] != b.shape[0]:
                    raise ShapeError("MPO bond mismatch between neighboring tensors")

    def __len__(self):
        return len(self.tensors)

    def __getitem__(self, n):
        return self.tensors[n]

    def bond_dimensions(self):
        return [self.tensors[0].shape[0]] + [t.shape[3] for t in self.tensors]

    def scaled(self, factor):  # mpo.hpp:54-74
        L = len(self)
        mag = abs(factor)
        if mag == 0:
            return MPO([np.zeros_like(t) for t in self.tensors])
        root = mag ** (1.0 / L)
        phase = factor / mag
        return MPO([t.astype(np.complex128) * (root * (phase if n == 0 else 1.0)) for n, t in enumerate(self.tensors)])


# ----------------------------------------------------------------------------
# truncated split (schmidt.hpp:18-94)
# ----------------------------------------------------------------------------


def svd_with_retry(theta: np.ndarray):
    """schmidt.hpp:18-36 (Eigen JacobiSVD thin -> LAPACK gesvd, gesdd fallback).
    Returns (U, s, Vh) with theta = U diag(s) Vh."""

    def run(m):
        try:
            return scipy.linalg.svd(m, full_matrices=False, lapack_driver="gesvd", check_finite=False)
        except np.linalg.LinAlgError:
            return scipy.linalg.svd(m, full_matrices=False, lapack_driver="gesdd", check_finite=False)

    def finite(r):
        return all(np.all(np.isfinite(x)) for x in r)

    try:
        out = run(theta)
        if finite(out):
            return out
    except np.linalg.LinAlgError:
        pass
    jit = theta.astype(np.complex128).copy()
    eps = 1e-14 * np.linalg.norm(theta)
    i = np.arange(theta.shape[0])[:, None]
    j = np.arange(theta.shape[1])[None, :]
    jit += eps * ((((i + 31 * j) % 7) / 7.0) + 1j * (((3 * i + j) % 5) / 5.0))
    try:
        out = run(jit)
        if finite(out):
            return out
    except np.linalg.LinAlgError:
        pass
    raise NumericError("SVD failed to converge after jitter retry")


def truncation_rank(s: np.ndarray, strategy: Strategy) -> int:
    """schmidt.hpp:40-52: strict `>` cutoff, at least 1, at most max_bond."""
    if s.size == 0:
        return 0
    cutoff = strategy.tolerance * s[0]
    rank = int(np.count_nonzero(s > cutoff))  # s is sorted descending
    rank = max(rank, 1)
    if strategy.max_bond != UNBOUNDED_BOND:
        rank = min(rank, strategy.max_bond)
    return rank


def dropped_weight(s: np.ndarray, rank: int) -> float:
    """schmidt.hpp:54-59."""
    return float(math.sqrt(float(np.sum(s[rank:] ** 2))))


def schmidt_split(theta: np.ndarray, strategy: Strategy, direction=LEFT_TO_RIGHT):
    """schmidt.hpp:72-89. Returns (a, b, error)."""
    if not np.all(np.isfinite(theta)):
        raise NumericError("schmidt_split: non-finite input")
    u, s, vh = svd_with_retry(theta)
    rank = truncation_rank(s, strategy)
    err = dropped_weight(s, rank)
    if GAP_LOG is not None and rank < s.size and s[rank - 1] > 0:
        GAP_LOG.append((theta.shape[0], theta.shape[1], rank, float(s[rank - 1]), float(s[rank]),
                        float((s[rank - 1] - s[rank]) / s[rank - 1])))
    if direction == LEFT_TO_RIGHT:
        return u[:, :rank], s[:rank, None] * vh[:rank], err
    return u[:, :rank] * s[None, :rank], vh[:rank], err


def schmidt_values(theta: np.ndarray) -> np.ndarray:
    """schmidt.hpp:92-94."""
    return svd_with_retry(theta)[1]


def split_pair(joined, d1, d2, strategy, direction):
    """mps.hpp:164-173."""
    al, dd, ar = joined.shape
    if dd != d1 * d2:
        raise ShapeError("split_pair: fused physical dimension mismatch")
    a, b, err = schmidt_split(joined.reshape(al * d1, d2 * ar), strategy, direction)
    rank = a.shape[1]
    return a.reshape(al, d1, rank), b.reshape(rank, d2, ar), err


def join_pair(a, b):
    """mps.hpp:148-155."""
    out = a.reshape(-1, a.shape[2]) @ b.reshape(b.shape[0], -1)
    return out.reshape(a.shape[0], a.shape[1] * b.shape[1], b.shape[2])


# ----------------------------------------------------------------------------
# environments (environments.hpp:13-37) and forms (forms.hpp:13-32)
# ----------------------------------------------------------------------------


def update_left_environment(env, bra, ket):
    """environments.hpp:18-23: E'[a',b'] = sum conj(A[a,s,a']) E[a,b] B[b,s,b']."""
    x = np.tensordot(env, ket, axes=([1], [0]))  # (a, s, b')
    return np.tensordot(bra.conj(), x, axes=([0, 1], [0, 1]))


def update_right_environment(env, bra, ket):
    """environments.hpp:26-31: E'[a,b] = sum conj(A[a,s,a']) E[a',b'] B[b,s,b']."""
    x = np.tensordot(ket, env, axes=([2], [1]))  # (b, s, a')
    return np.tensordot(bra.conj(), x, axes=([1, 2], [1, 2]))


def project_pair(lenv, k1, k2, renv):
    """forms.hpp:13-32, in the reference's order: the (B*d1) x (d2*B'') pair
    product first, then L * blk * R^T for each (i1, i2)."""
    d1, d2 = k1.shape[1], k2.shape[1]
    pair = k1.reshape(-1, k1.shape[2]) @ k2.reshape(k2.shape[0], -1)
    pair = pair.reshape(k1.shape[0], d1, d2, k2.shape[2])
    out = np.empty((lenv.shape[0], d1 * d2, renv.shape[0]), dtype=np.result_type(lenv, pair, renv))
    for i1 in range(d1):
        for i2 in range(d2):
            out[:, i1 * d2 + i2, :] = lenv @ pair[:, i1, i2, :] @ renv.T
    return out


def project_pair_fast(lenv, k1, k2, renv):
    """Same value as project_pair in the minimal-flop order (L*T1)*T2*R^T."""
    x = np.tensordot(lenv, k1, axes=([1], [0]))  # (a, i1, B')
    y = np.tensordot(x, k2, axes=([2], [0]))  # (a, i1, i2, B'')
    f = np.tensordot(y, renv, axes=([3], [1]))  # (a, i1, i2, b)
    return f.reshape(f.shape[0], f.shape[1] * f.shape[2], f.shape[3])


def scprod(u: MPS, v: MPS):
    """mps.hpp:416-423."""
    if len(u) != len(v):
        raise ShapeError("scprod: states of different length")
    env = np.ones((1, 1), dtype=np.result_type(u[0], v[0]))
    for a, b in zip(u.tensors, v.tensors):
        env = update_left_environment(env, a, b)
    return env[0, 0]


def mps_to_dense(state: MPS, guard=DENSE_VECTOR_GUARD) -> np.ndarray:
    """mps.hpp:438-449 (most significant site first)."""
    dim = state.dimension(guard)
    acc = np.ones((1, 1), dtype=state[0].dtype)
    for t in state.tensors:
        nxt = acc @ t.reshape(t.shape[0], -1)
        acc = nxt.reshape(-1, t.shape[2])
    if acc.shape != (dim, 1):
        raise ShapeError("mps_to_dense: inconsistent contraction")
    return acc[:, 0]


# ----------------------------------------------------------------------------
# simplification engine (simplify.hpp:15-195)
# ----------------------------------------------------------------------------


class CompressionEngine:
    """simplify.hpp:15-92 for a single term with weight 1 (simplify(MPS))."""

    def __init__(self, weights, states, guess: MPS, strategy: Strategy, fast=False):
        self.weights = list(weights)
        self.states = list(states)
        self.fast = fast
        self.psi = CanonicalMPS(guess, 0, strategy.with_normalize(False))  # simplify.hpp:25
        L = len(self.psi)
        dt = np.result_type(self.psi[0], *[s[0] for s in self.states])
        one = np.ones((1, 1), dtype=dt)
        self.lenv = [[None] * (L + 1) for _ in self.states]
        self.renv = [[None] * (L + 1) for _ in self.states]
        for l, st in enumerate(self.states):  # simplify.hpp:30-36
            self.lenv[l][0] = one
            self.renv[l][L] = one
            for n in range(L - 1, 0, -1):
                self.renv[l][n] = update_right_environment(self.renv[l][n + 1], self.psi[n], st[n])
        acc = 0.0  # simplify.hpp:37-41
        for l, sl in enumerate(self.states):
            for m, sm in enumerate(self.states):
                acc += np.conj(self.weights[l]) * self.weights[m] * scprod(sl, sm)
        self.target_norm2 = max(0.0, float(np.real(acc)))

    def projected_pair(self, n):  # simplify.hpp:44-62
        proj = project_pair_fast if self.fast else project_pair
        out = None
        for l, st in enumerate(self.states):
            f = self.weights[l] * proj(self.lenv[l][n], st[n], st[n + 1], self.renv[l][n + 2])
            if np.iscomplexobj(f) and not np.iscomplexobj(st[n]) and np.all(f.imag == 0):
                f = f.real
            out = f if out is None else out + f
        return out

    def sweep(self, strategy) -> float:  # simplify.hpp:66-91
        psi = self.psi
        L = len(psi)
        if L == 1:
            t = sum(self.weights[l] * st[0] for l, st in enumerate(self.states))
            psi.tensors[0] = t
            return max(0.0, self.target_norm2 - psi.norm_squared())
        psi.recenter(0, strategy)
        for n in range(L - 1):
            psi.update_two_site(self.projected_pair(n), LEFT_TO_RIGHT, strategy)
            for l, st in enumerate(self.states):
                self.lenv[l][n + 1] = update_left_environment(self.lenv[l][n], psi[n], st[n])
        for n in range(L - 2, -1, -1):
            psi.update_two_site(self.projected_pair(n), RIGHT_TO_LEFT, strategy)
            for l, st in enumerate(self.states):
                self.renv[l][n + 1] = update_right_environment(self.renv[l][n + 2], psi[n + 1], st[n + 1])
        return max(0.0, self.target_norm2 - psi.norm_squared())


@dataclass
class CompressionResult:
    state: CanonicalMPS
    residual: float = 0.0
    sweeps: int = 0
    converged: bool = False
    dist2_history: Optional[list] = None
    target_norm2: float = 0.0


def variational_compress(weights, states, guess, strategy, fast=False, max_steps=None) -> CompressionResult:
    """simplify.hpp:101-131."""
    engine = CompressionEngine(weights, states, guess, strategy, fast=fast)
    target_norm = math.sqrt(engine.target_norm2)
    if target_norm <= fp_error_floor(1.0):
        return CompressionResult(CanonicalMPS(states[0].zero_like(), 0, NO_TRUNCATION), target_norm, 0, True, [],
                                 engine.target_norm2)
    out = CompressionResult(None, 0.0, 0, False, [], engine.target_norm2)
    dist2 = engine.target_norm2
    sweeps = max(1, strategy.max_sweeps) if max_steps is None else max_steps
    for sweep in range(sweeps):
        prev = dist2
        dist2 = engine.sweep(strategy)
        out.sweeps += 1
        out.dist2_history.append(dist2)
        if math.sqrt(dist2) <= strategy.simplification_tolerance * target_norm:  # simplify.hpp:118
            out.converged = True
            break
        if sweep > 0 and abs(prev - dist2) <= 1e-15 * engine.target_norm2:  # simplify.hpp:123
            break
    out.residual = math.sqrt(max(0.0, dist2)) + fp_error_floor(target_norm)  # simplify.hpp:126
    out.state = engine.psi
    if out.state.norm() == 0.0:
        out.state = CanonicalMPS(states[0].zero_like(), 0, NO_TRUNCATION)
    return out


def simplify(target: MPS, strategy: Strategy = DEFAULT_STRATEGY, guess: Optional[MPS] = None, *, promote=False,
             fast=False, report: Optional[dict] = None) -> CanonicalMPS:
    """simplify.hpp:182-195."""
    if promote:
        target = MPS([t.astype(np.complex128) for t in target.tensors], target.error)
    if strategy.method == SVD_TRUNCATE:
        return CanonicalMPS(target, 0, strategy)
    carried = target.error
    res = variational_compress([1.0], [target], guess if guess is not None else target, strategy, fast=fast)
    res.state.error = carried + res.residual
    if strategy.normalize:
        res.state.normalize_in_place()
    if report is not None:
        report.update(sweeps=res.sweeps, residual=res.residual, converged=res.converged,
                      dist2=res.dist2_history, target_norm2=res.target_norm2)
    return res.state


class MPSSum:
    """mps.hpp:326-412: lazy weighted sum of states with equal physical dimensions."""

    def __init__(self, weights, states):
        weights, states = list(weights), list(states)
        if not weights or len(weights) != len(states):
            raise ShapeError("MPSSum: weights and states must be non-empty and match")
        dims = states[0].physical_dimensions()
        for st in states:
            if st.physical_dimensions() != dims:
                raise ShapeError("MPSSum: states must share physical dimensions")
        self.weights, self.states = weights, states

    def error(self) -> float:  # mps.hpp:344-349
        return float(sum(abs(w) * st.error for w, st in zip(self.weights, self.states)))

    def join(self) -> MPS:  # mps.hpp:352-405
        scaled = [st.scaled(w) for w, st in zip(self.weights, self.states)]
        if len(scaled) == 1:
            return scaled[0]
        L = len(scaled[0])
        cplx = any(np.iscomplexobj(t) for sc in scaled for t in sc.tensors)
        dt = np.complex128 if cplx else np.float64
        out = []
        for n in range(L):
            dl = sum(sc[n].shape[0] for sc in scaled)
            dr = sum(sc[n].shape[2] for sc in scaled)
            d = scaled[0][n].shape[1]
            if n == 0:
                t = np.zeros((1, d, dr), dtype=dt)
                off = 0
                for sc in scaled:
                    b = sc[n].shape[2]
                    t[0, :, off:off + b] = sc[n][0]
                    off += b
            elif n == L - 1:
                t = np.zeros((dl, d, 1), dtype=dt)
                off = 0
                for sc in scaled:
                    a = sc[n].shape[0]
                    t[off:off + a, :, 0] = sc[n][:, :, 0]
                    off += a
            else:
                t = np.zeros((dl, d, dr), dtype=dt)
                ol = orr = 0
                for sc in scaled:
                    a, _, b = sc[n].shape
                    t[ol:ol + a, :, orr:orr + b] = sc[n]
                    ol += a
                    orr += b
            out.append(t)
        return MPS(out, self.error())


def default_guess(weights, states) -> MPS:
    """simplify.hpp:133-144."""
    best, bw = 0, -1.0
    for l, st in enumerate(states):
        w = abs(weights[l]) * st.norm()
        if w > bw:
            best, bw = l, w
    return states[best].scaled(weights[best])


def simplify_sum(target: MPSSum, strategy: Strategy = DEFAULT_STRATEGY, guess: Optional[MPS] = None,
                 report: Optional[dict] = None) -> CanonicalMPS:
    """simplify.hpp:198-215 (simplify(MPSSum))."""
    if strategy.method == SVD_TRUNCATE:
        out = CanonicalMPS(target.join(), 0, strategy.with_normalize(False))
        if strategy.normalize:
            out.normalize_in_place()
        return out
    carried = target.error()
    res = variational_compress(target.weights, target.states,
                               guess if guess is not None else default_guess(target.weights, target.states),
                               strategy)
    res.state.error = carried + res.residual
    if strategy.normalize:
        res.state.normalize_in_place()
    if report is not None:
        report.update(sweeps=res.sweeps, residual=res.residual, converged=res.converged,
                      dist2=res.dist2_history, target_norm2=res.target_norm2)
    return res.state


def combine(weights, states, strategy=DEFAULT_STRATEGY) -> CanonicalMPS:
    """simplify.hpp:151-179."""
    weights, states = list(weights), list(states)
    if not weights or len(weights) != len(states):
        raise ShapeError("combine: weights and states must be non-empty and match")
    dims = states[0].physical_dimensions()
    for st in states:
        if st.physical_dimensions() != dims:
            raise ShapeError("combine: states must share physical dimensions")
    carried = sum(abs(w) * st.error for w, st in zip(weights, states))
    if strategy.method == SVD_TRUNCATE:
        joined = MPSSum(weights, states).join()
        out = CanonicalMPS(joined, 0, strategy.with_normalize(False))
        out.error = out.error - joined.error
    else:
        res = variational_compress(weights, states, default_guess(weights, states), strategy)
        out = res.state
        out.error = res.residual
    out.error = carried + out.error
    if strategy.normalize:
        out.normalize_in_place()
    return out


# ----------------------------------------------------------------------------
# expansions (mpo.hpp:213-238, blas.hpp:8-11, 45-67)
# ----------------------------------------------------------------------------


def apply_raw(op: MPO, v: MPS) -> MPS:
    """mpo.hpp:213-238: C[(cb*chi_l+al), j, (cb2*chi_r+ar)] = sum_i W[cb,j,i,cb2] A[al,i,ar]."""
    if len(op) != len(v):
        raise ShapeError("apply: operator and state sizes differ")
    out = []
    for w, a in zip(op.tensors, v.tensors):
        if w.shape[2] != a.shape[1]:
            raise ShapeError("apply: physical dimension mismatch")
        c = np.einsum("cjid,aib->cajdb", w, a)
        out.append(c.reshape(w.shape[0] * a.shape[0], w.shape[1], w.shape[3] * a.shape[2]))
    return MPS(out, v.error)


def apply(op: MPO, v: MPS, strategy: Strategy = DEFAULT_STRATEGY, **kw) -> CanonicalMPS:
    """blas.hpp:8-11."""
    return simplify(apply_raw(op, v), strategy, **kw)


def apply_sum(op: MPO, v: MPSSum, strategy: Strategy = DEFAULT_STRATEGY) -> CanonicalMPS:
    """blas.hpp:13-20."""
    return simplify_sum(MPSSum(v.weights, [apply_raw(op, st) for st in v.states]), strategy)


def apply_list(ops: Sequence[MPO], v, strategy: Strategy = DEFAULT_STRATEGY) -> CanonicalMPS:
    """blas.hpp:24-42: factors applied last entry first; v an MPS or an MPSSum."""
    if len(ops) == 0:
        raise ShapeError("apply: empty MPO list")
    state = apply_sum(ops[-1], v, strategy) if isinstance(v, MPSSum) else apply(ops[-1], v, strategy)
    for k in range(len(ops) - 2, -1, -1):
        state = apply(ops[k], state, strategy)
    return state


def hadamard(u: MPS, v: MPS) -> MPS:
    """blas.hpp:45-67: C[(a*chi_b+b), s, (a'*chi_b'+b')] = A[a,s,a'] B[b,s,b']."""
    if len(u) != len(v):
        raise ShapeError("hadamard: states of different length")
    out = []
    for a, b in zip(u.tensors, v.tensors):
        if a.shape[1] != b.shape[1]:
            raise ShapeError("hadamard: physical dimension mismatch")
        c = np.einsum("asc,bsd->abscd", a, b)
        out.append(c.reshape(a.shape[0] * b.shape[0], a.shape[1], a.shape[2] * b.shape[2]))
    return MPS(out, u.error + v.error)


# ----------------------------------------------------------------------------
# constructors used by the pins (mps.hpp:493-544, mpo.hpp:132-207, 273-312)
# ----------------------------------------------------------------------------


def random_uniform_mps(L, d, bond, seed) -> MPS:
    """mps.hpp:493-514 (bit-exact under libstdc++; see oracle/rng.py)."""
    from .rng import MT19937_64, complex_draws

    if L < 1 or d < 1 or bond < 1:
        raise ShapeError("random_uniform_mps: L, d, bond must be >= 1")
    rng = MT19937_64(seed)

    def bond_at(cut):
        cap = min(float(bond), float(d) ** cut, float(d) ** (L - cut))
        return int(max(1.0, cap))

    ts = []
    for n in range(L):
        shape = (bond_at(n), d, bond_at(n + 1))
        ts.append(complex_draws(rng, int(np.prod(shape))).reshape(shape))
    return MPS(ts, 0.0)


def product_state(L, site) -> MPS:
    site = np.asarray(site, dtype=np.complex128)
    return MPS([site.reshape(1, -1, 1).copy() for _ in range(L)])


def basis_state(L, d, idx) -> MPS:
    """mps.hpp:530-544 (most significant first)."""
    ts = []
    rem = idx
    for _ in range(L):
        t = np.zeros((1, d, 1), dtype=np.complex128)
        t[0, rem % d, 0] = 1.0
        ts.append(t)
        rem //= d
    return MPS(ts[::-1])


def mpo_identity(L, d) -> MPO:
    """mpo.hpp:132-144."""
    return MPO([np.eye(d, dtype=np.complex128).reshape(1, d, d, 1) for _ in range(L)])


def mpo_from_local_operators(ops) -> MPO:
    """mpo.hpp:158-169."""
    return MPO([np.asarray(m, dtype=np.complex128).reshape(1, m.shape[0], m.shape[1], 1) for m in ops])


def mpo_sum(weights, terms) -> MPO:
    """mpo.hpp:273-312 (block concatenation)."""
    if not weights or len(weights) != len(terms):
        raise ShapeError("mpo_sum: weights and terms must be non-empty and match")
    if len(terms) == 1:
        return terms[0].scaled(weights[0])
    sc = [t.scaled(w) for w, t in zip(weights, terms)]
    L = len(terms[0])
    out = []
    for n in range(L):
        dl = sum(t[n].shape[0] for t in sc)
        dr = sum(t[n].shape[3] for t in sc)
        first, last = n == 0, n == L - 1
        do, di = sc[0][n].shape[1], sc[0][n].shape[2]
        t = np.zeros((1 if first else dl, do, di, 1 if last else dr), dtype=np.complex128)
        ol = orr = 0
        for term in sc:
            b = term[n]
            sl = slice(0, 1) if first else slice(ol, ol + b.shape[0])
            sr = slice(0, 1) if last else slice(orr, orr + b.shape[3])
            t[sl, :, :, sr] += b
            ol += b.shape[0]
            orr += b.shape[3]
        out.append(t)
    return MPO(out)


def mpo_to_dense(op: MPO, guard=DENSE_OPERATOR_GUARD) -> np.ndarray:
    """mpo.hpp:172-207 (row index = output, earlier sites most significant)."""
    jd = idim = 1
    for t in op.tensors:
        jd *= t.shape[1]
        idim *= t.shape[2]
        if jd > guard or idim > guard:
            raise CapacityError("mpo_to_dense: dimension exceeds guard")
    acc = [np.ones((1, 1), dtype=np.complex128)]
    for t in op.tensors:
        nxt = []
        for b in range(t.shape[3]):
            m = 0
            for a in range(t.shape[0]):
                m = m + np.kron(acc[a], t[a, :, :, b])
            nxt.append(m)
        acc = nxt
    if len(acc) != 1:
        raise ShapeError("mpo_to_dense: unclosed bond")
    return acc[0]


def shift_mpo(n, m, periodic=True) -> MPO:
    """shifts.hpp:16-45 (binary adder with a carry bond of two); used only to
    cross-check the Laplacian MPO of config 2."""
    size = 1 << n
    m_mod = ((m % size) + size) % size
    if m_mod == 0 and (periodic or m == 0):
        return mpo_identity(n, 2)
    required = 1 if (not periodic and m < 0) else 0
    ts = []
    for site in range(n):
        bit = n - 1 - site
        mbit = (m_mod >> bit) & 1
        right = 1 if site == n - 1 else 2
        left = 1 if site == 0 else 2
        t = np.zeros((left, 2, 2, right), dtype=np.complex128)
        for cin in range(1 if site == n - 1 else 2):
            for o in range(2):
                i = o ^ mbit ^ cin
                cout = (o + mbit + cin) >> 1
                if site == 0:
                    if periodic or cout == required:
                        t[0, o, i, cin] = 1.0
                else:
                    t[cout, o, i, 0 if site == n - 1 else cin] = 1.0
        ts.append(t)
    return MPO(ts)


# ----------------------------------------------------------------------------
# Fourier transform (qft.hpp:10-128), restated as dense circuits
# ----------------------------------------------------------------------------


def qft_layer_dense(L, sites, m, sign, carry_input) -> np.ndarray:
    """qft.hpp:10-15 as a dense 2^L x 2^L matrix: Hadamard on qubit sites[m]
    (site 0 most significant) and, for every later subset qubit sites[j],
    the phase exp(i sign 2 pi c b_j / 2^(j-m+1)) with c the Hadamard's output
    bit (forward layer: phases after H) or input bit (adjoint layer: phases
    before H)."""
    dim = 1 << L
    bit = lambda x, q: (x >> (L - 1 - q)) & 1

    def phase(c_of):
        ph = np.ones(dim, dtype=np.complex128)
        for x in range(dim):
            c = c_of(x)
            for j in range(m + 1, len(sites)):
                ph[x] *= np.exp(1j * sign * 2.0 * np.pi * c * bit(x, sites[j]) / 2.0 ** (j - m + 1))
        return np.diag(ph)

    h = np.array([[1.0, 1.0], [1.0, -1.0]]) / np.sqrt(2.0)
    q = sites[m]
    H = np.kron(np.kron(np.eye(1 << q), h), np.eye(1 << (L - 1 - q)))
    P = phase(lambda x: bit(x, q))
    return H @ P if carry_input else P @ H


def qft_dense(L, inverse=False, sites=None) -> np.ndarray:
    """qft.hpp:67-101: product of the layers (forward: layer 0 acts first;
    inverse: the conjugated layers in the opposite order)."""
    subset = list(range(L)) if sites is None else list(sites)
    sign = 1.0 if inverse else -1.0
    order = range(len(subset) - 1, -1, -1) if inverse else range(len(subset))
    U = np.eye(1 << L, dtype=np.complex128)
    for m in order:
        U = qft_layer_dense(L, subset, m, sign, inverse) @ U
    return U


def bit_reversal(L) -> np.ndarray:
    """qft.hpp:114-126 (qft_flip) as a permutation matrix."""
    dim = 1 << L
    P = np.zeros((dim, dim))
    for x in range(dim):
        P[int(format(x, f"0{L}b")[::-1], 2), x] = 1.0
    return P


# ----------------------------------------------------------------------------
# operator environments and expectation values (environments.hpp:38-89,
# blas.hpp:100-138)
# ----------------------------------------------------------------------------


def update_left_op_environment(env, bra, op, ket):
    """environments.hpp:45-63: E'[c'](a',b') = sum conj(A[a,s',a']) W[c,s',s,c'] E[c](a,b) B[b,s,b'].
    env has shape (c, a, b)."""
    return np.einsum("cab,axy,cxsd,bsz->dyz", env, np.conj(bra), op, ket, optimize=True)


def update_right_op_environment(env, bra, op, ket):
    """environments.hpp:67-83: E'[c](a,b) = sum conj(A[a,s',a']) W[c,s',s,c'] E[c'](a',b') B[b,s,b'].
    env has shape (c', a', b')."""
    return np.einsum("dyz,axy,cxsd,bsz->cab", env, np.conj(bra), op, ket, optimize=True)


def apply_effective_two_site(lenv, w1, w2, renv, x):
    """eigensolvers.hpp:15-64 detail::apply_effective_two_site, step for step: X[c0] = L[c0] x
    (:30-33), the W1 contraction into T[c1] (:34-46), the W2 contraction into U[c2] (:47-59), then
    y = sum_c2 U[c2] R[c2]^T (:60-63).  lenv (D0, chiAo, chiA), renv (D2, chiBo, chiB)."""
    L, R = np.asarray(lenv), np.asarray(renv)
    w1, w2 = np.asarray(w1), np.asarray(w2)
    chiAo, chiA = L.shape[1:]
    chiBo, chiB = R.shape[1:]
    D0, d1o, d1, D1 = w1.shape
    _, d2o, d2, D2 = w2.shape
    x = np.asarray(x).reshape(-1)
    if x.size != chiA * d1 * d2 * chiB:
        raise ShapeError("apply_effective_two_site: bad vector size")
    xmat = x.reshape(chiA, d1 * d2 * chiB)
    xl = [L[c0] @ xmat for c0 in range(D0)]
    t = [np.zeros((chiAo * d1o, d2 * chiB), dtype=np.complex128) for _ in range(D1)]
    for c0 in range(D0):
        for s1o in range(d1o):
            for s1 in range(d1):
                for c1 in range(D1):
                    w = w1[c0, s1o, s1, c1]
                    if w == 0:
                        continue
                    for a in range(chiAo):
                        t[c1][a * d1o + s1o] += w * xl[c0][a, s1 * d2 * chiB:(s1 + 1) * d2 * chiB]
    u = [np.zeros((chiAo * d1o * d2o, chiB), dtype=np.complex128) for _ in range(D2)]
    for c1 in range(D1):
        for s2o in range(d2o):
            for s2 in range(d2):
                for c2 in range(D2):
                    w = w2[c1, s2o, s2, c2]
                    if w == 0:
                        continue
                    for row in range(chiAo * d1o):
                        u[c2][row * d2o + s2o] += w * t[c1][row, s2 * chiB:(s2 + 1) * chiB]
    y = np.zeros((chiAo * d1o * d2o, chiBo), dtype=np.complex128)
    for c2 in range(D2):
        y += u[c2] @ R[c2].T
    return y.reshape(-1)


def expectation_mpo(op: MPO, u: MPS, v: Optional[MPS] = None):
    """blas.hpp:128-138."""
    ket = v if v is not None else u
    if len(op) != len(u) or len(ket) != len(u):
        raise ShapeError("expectation_mpo: size mismatch")
    env = np.ones((1, 1, 1), dtype=np.complex128)
    for n in range(len(u)):
        env = update_left_op_environment(env, u[n], op[n], ket[n])
    if env.shape[0] != 1:
        raise ShapeError("expectation_mpo: unclosed MPO bond")
    return complex(env[0, 0, 0])


def expectation_local(v: MPS, op, site, op2=None, site2=None):
    """blas.hpp:100-125: <v, O_site v> or <v, O_site O2_site2 v> (bra/ket environment chain)."""
    if site < 0 or site >= len(v):
        raise ShapeError("expectation_local: site out of range")
    if (op2 is None) != (site2 is None):
        raise ShapeError("expectation_local: two-point value needs both operator and site")
    if op2 is not None and (site2 < 0 or site2 >= len(v) or site2 == site):
        raise ShapeError("expectation_local: second site out of range")
    env = np.ones((1, 1), dtype=np.complex128)
    for n in range(len(v)):
        ket = v[n]
        for o, k in ((op, site), (op2, site2)):
            if o is not None and n == k and np.shape(o) != (ket.shape[1], ket.shape[1]):
                raise ShapeError("local operator dimension mismatch")  # blas.hpp:88-89
        if n == site:
            ket = np.einsum("ts,asb->atb", op, ket)
        if op2 is not None and n == site2:
            ket = np.einsum("ts,asb->atb", op2, ket)
        env = update_left_environment(env, v[n], ket)
    return complex(env[0, 0])


# ----------------------------------------------------------------------------
# TTLAB1 container (serialize.hpp:13-121)
# ----------------------------------------------------------------------------

TTLAB_MAGIC = b"TTLAB1\0"


def _write_tensor(buf: list, t: np.ndarray):
    import struct
    buf.append(struct.pack("<B", t.ndim) + struct.pack("<" + "Q" * t.ndim, *t.shape))
    buf.append(np.ascontiguousarray(t, dtype="<c16").tobytes())


def dumps_mps(state: MPS) -> bytes:
    """serialize.hpp:67-80."""
    import struct
    buf = [TTLAB_MAGIC, struct.pack("<II", 1, len(state))]
    for t in state.tensors:
        _write_tensor(buf, t)
    buf.append(struct.pack("<d", state.error))
    return b"".join(buf)


def dumps_mpo(op: MPO) -> bytes:
    """serialize.hpp:101-112."""
    import struct
    buf = [TTLAB_MAGIC, struct.pack("<II", 1, len(op))]
    for t in op.tensors:
        _write_tensor(buf, t)
    return b"".join(buf)


def _reader(data: bytes):
    import struct
    pos = [0]

    def take(n):
        if pos[0] + n > len(data):
            raise NumericError("ttlab container: truncated file")
        out = data[pos[0]:pos[0] + n]
        pos[0] += n
        return out

    def header():
        if take(7) != TTLAB_MAGIC:
            raise NumericError("ttlab container: bad magic")
        version, count = struct.unpack("<II", take(8))
        if version != 1:
            raise NumericError("ttlab container: unsupported version")
        return count

    def tensor(rank):
        if struct.unpack("<B", take(1))[0] != rank:
            raise NumericError(f"ttlab container: expected rank-{rank} tensor")
        dims = struct.unpack("<" + "Q" * rank, take(8 * rank))
        n = int(np.prod(dims))
        return np.frombuffer(take(16 * n), dtype="<c16").reshape(dims).astype(np.complex128)

    return take, header, tensor


def loads_mps(data: bytes) -> MPS:
    """serialize.hpp:82-99."""
    import struct
    take, header, tensor = _reader(data)
    ts = [tensor(3) for _ in range(header())]
    return MPS(ts, struct.unpack("<d", take(8))[0])


def loads_mpo(data: bytes) -> MPO:
    """serialize.hpp:114-130."""
    _, header, tensor = _reader(data)
    return MPO([tensor(4) for _ in range(header())])
