"""Bounded CPU timing of one full apply/simplify call in reference arithmetic.

TEST / BENCH INFRASTRUCTURE (the `cpu_baseline` leg and `bench.py --impl
reference`): never imported by the product package.

A full C3/C4 call of the CPU restatement takes many minutes on the host (the
reference forms every two-site pair first, forms.hpp:18, and promotes to
complex128, types.hpp:12-16).  This module times it as a sum of *units*, the
pieces the reference executes one after the other:

  qr    site k of the exact left-to-right pass (mps.hpp:193-205):
        Householder QR of the (q_k d x t_{k+1}) unfolding + carry R T_{k+1}
  trunc site k of the truncating right-to-left pass (mps.hpp:206-210, 253-265):
        SVD of the (q_k x d p_{k+1}) centre + carry of U S into site k-1
  renv  right environment k (simplify.hpp:30-36, environments.hpp:26-31)
  norm  one step of scprod(T, T) (simplify.hpp:37-41, mps.hpp:416-423)
  step  one two-site step of a sweep (simplify.hpp:66-91): pair-first
        project_pair (forms.hpp:13-32) + schmidt_split + environment update

The unit list and every unit's shape follow from the bond recursion alone
(target bonds t, exact-pass bonds q, output bonds p).  Units of identical shape
cost the same, so they are grouped; `measure(budget)` times one representative
of the next groups (largest estimated work first, random complex128 operands
of the exact shapes: dense LAPACK/BLAS cost does not depend on the values) and
`estimate()` returns the full-call time = sum over groups of count x measured
time, where groups not measured yet are extrapolated from the measured rate
(flop/s) of their own unit kind.  `coverage()` says which fraction of the
estimated work was measured directly.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import ttlab_oracle as O


@dataclass
class Group:
    kind: str
    shape: Tuple[int, ...]
    count: int
    flops: float  # estimated real flops of ONE unit in reference arithmetic
    times: List[float] = field(default_factory=list)


def _zgemm(m, n, k):
    return 8.0 * m * n * k


def _zqr(m, n):  # Householder R + explicit thin Q, complex
    a, b = max(m, n), min(m, n)
    return 4.0 * 4.0 * b * b * (a - b / 3.0)


def _zsvd(m, n):  # Golub-Van Loan R-SVD with U and V, complex
    a, b = max(m, n), min(m, n)
    return 4.0 * (4 * a * a * b + 8 * a * b * b + 9 * b * b * b)


def units(t: Sequence[int], p: Sequence[int], d: Sequence[int], sweeps: int, norm_chain: bool = True) -> List[Group]:
    """Group the units of one call.  t: target bonds (L+1), p: output bonds (L+1), d: (L)."""
    L = len(d)
    q = [1] * (L + 1)
    for k in range(L - 1):
        q[k + 1] = min(q[k] * d[k], t[k + 1])
    groups: Dict[Tuple, Group] = {}

    def add(kind, shape, flops, count=1):
        key = (kind,) + tuple(shape)
        if key not in groups:
            groups[key] = Group(kind, tuple(shape), 0, flops)
        groups[key].count += count

    for k in range(L - 1):
        m, n = q[k] * d[k], t[k + 1]
        add("qr", (m, n, min(m, n), d[k + 1] * t[k + 2]),
            _zqr(m, n) + _zgemm(min(m, n), d[k + 1] * t[k + 2], n))
    for k in range(L - 1, 0, -1):
        m, n = q[k], d[k] * p[k + 1]
        r = p[k]
        add("trunc", (m, n, r, q[k - 1] * d[k - 1]), _zsvd(m, n) + _zgemm(q[k - 1] * d[k - 1], r, m))
    for k in range(L - 1, 0, -1):
        add("renv", (t[k], d[k], t[k + 1], p[k], p[k + 1]),
            _zgemm(t[k] * d[k], p[k + 1], t[k + 1]) + _zgemm(p[k], t[k], d[k] * p[k + 1]))
    if norm_chain:
        for k in range(L):
            add("norm", (t[k], d[k], t[k + 1]), _zgemm(t[k], d[k] * t[k + 1], t[k]) + _zgemm(t[k + 1], t[k + 1], t[k] * d[k]))
    for _ in range(sweeps):
        for direction in (O.LEFT_TO_RIGHT, O.RIGHT_TO_LEFT):
            for n in range(L - 1):
                dn, dn1 = d[n], d[n + 1]
                pair = _zgemm(t[n] * dn, dn1 * t[n + 2], t[n + 1])
                proj = dn * dn1 * (_zgemm(p[n], t[n + 2], t[n]) + _zgemm(p[n], p[n + 2], t[n + 2]))
                split = _zsvd(p[n] * dn, dn1 * p[n + 2])
                env = _zgemm(p[n] * dn, t[n + 1], t[n]) + _zgemm(p[n + 1], t[n + 1], p[n] * dn)
                add("step", (p[n], t[n], dn, t[n + 1], dn1, t[n + 2], p[n + 2], p[n + 1], int(direction)),
                    pair + proj + split + env)
    return sorted(groups.values(), key=lambda g: -g.count * g.flops)


def _rand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def run_unit(g: Group, rng) -> float:
    """Execute one unit of group g with the oracle's reference-arithmetic code; returns seconds."""
    s = g.shape
    strat = O.Strategy(max_bond=O.UNBOUNDED_BOND, tolerance=1e-12)
    if g.kind == "qr":
        m, n, r, nxt = s
        a, b = _rand(rng, m, n), _rand(rng, n, nxt)
        t0 = time.perf_counter()
        qm, rm = np.linalg.qr(a, mode="reduced")
        _ = rm @ b
        return time.perf_counter() - t0
    if g.kind == "trunc":
        m, n, r, prev_rows = s
        theta, prev = _rand(rng, m, n), _rand(rng, prev_rows, m)
        t0 = time.perf_counter()
        u, sv, vh = O.svd_with_retry(theta)
        us = u[:, :r] * sv[None, :r]
        _ = prev @ us
        return time.perf_counter() - t0
    if g.kind == "renv":
        tk, dk, tk1, pk, pk1 = s
        env, psi, tt = _rand(rng, pk1, tk1), _rand(rng, pk, dk, pk1), _rand(rng, tk, dk, tk1)
        t0 = time.perf_counter()
        O.update_right_environment(env, psi, tt)
        return time.perf_counter() - t0
    if g.kind == "norm":
        tk, dk, tk1 = s
        env, tt = _rand(rng, tk, tk), _rand(rng, tk, dk, tk1)
        t0 = time.perf_counter()
        O.update_left_environment(env, tt, tt)
        return time.perf_counter() - t0
    if g.kind == "step":
        pn, tn, dn, tn1, dn1, tn2, pn2, pn1, direction = s
        lenv, renv = _rand(rng, pn, tn), _rand(rng, pn2, tn2)
        k1, k2 = _rand(rng, tn, dn, tn1), _rand(rng, tn1, dn1, tn2)
        t0 = time.perf_counter()
        f = O.project_pair(lenv, k1, k2, renv)
        st = O.Strategy(max_bond=max(1, pn1), tolerance=1e-12)
        a, b, _ = O.split_pair(f, dn, dn1, st, direction)
        if direction == O.LEFT_TO_RIGHT:
            O.update_left_environment(lenv, a, k1)
        else:
            O.update_right_environment(renv, b, k2)
        return time.perf_counter() - t0
    raise ValueError(g.kind)


class CallModel:
    """Full-call CPU time = sum over unit groups of count x time of one unit."""

    def __init__(self, t, p, d, sweeps, seed=0, norm_chain=True):
        self.groups = units(t, p, d, sweeps, norm_chain)
        self.rng = np.random.default_rng(seed)
        self._next = 0

    def measure(self, budget_s: float) -> int:
        """Time the next groups in the queue (largest work first, cyclic) for at
        least one unit and until `budget_s` seconds are used; returns units timed."""
        t0, done = time.perf_counter(), 0
        while done == 0 or time.perf_counter() - t0 < budget_s:
            g = self.groups[self._next % len(self.groups)]
            g.times.append(run_unit(g, self.rng))
            self._next += 1
            done += 1
            if self._next % len(self.groups) == 0 and time.perf_counter() - t0 >= budget_s:
                break
        return done

    def estimate(self) -> float:
        rate: Dict[str, Tuple[float, float]] = {}
        for g in self.groups:
            if g.times:
                f, s = rate.get(g.kind, (0.0, 0.0))
                rate[g.kind] = (f + g.flops, s + float(np.mean(g.times)))
        all_f = sum(v[0] for v in rate.values())
        all_s = sum(v[1] for v in rate.values())
        total = 0.0
        for g in self.groups:
            if g.times:
                total += g.count * float(np.mean(g.times))
            else:
                f, s = rate.get(g.kind, (all_f, all_s))
                total += g.count * g.flops * (s / f if f > 0 else 0.0)
        return total

    def coverage(self) -> float:
        tot = sum(g.count * g.flops for g in self.groups)
        return sum(g.count * g.flops for g in self.groups if g.times) / tot if tot else 1.0

    def units_timed(self) -> int:
        return sum(len(g.times) for g in self.groups)

    def total_units(self) -> int:
        return sum(g.count for g in self.groups)
