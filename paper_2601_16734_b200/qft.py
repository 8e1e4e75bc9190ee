"""Quantum Fourier transform as an MPO list (reference qft.hpp:10-128).

The layer MPOs are tiny host-side constructors (bond dimension <= 2); the
transform itself is `ttlab.apply(MPOList, state)`, i.e. one device
apply_raw + variational simplify per layer on the B200 (blas.hpp:24-42).

Conventions follow the reference: site 0 is the most significant qubit, the
forward transform leaves its output in bit-reversed order so that
`qft_flip(qft(v))` is the unitary DFT with kernel exp(-2 pi i jk / 2^n).
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from . import ttlab

_R2 = 1.0 / np.sqrt(2.0)


def _identity_site():
    t = np.zeros((1, 2, 2, 1), dtype=np.complex128)
    t[0, 0, 0, 0] = t[0, 1, 1, 0] = 1.0
    return t


def qft_layer(L: int, sites: Sequence[int], m: int, sign: float, carry_input: bool):
    """qft.hpp:16-60.  Hadamard on sites[m]; every later subset qubit q = sites[j]
    picks up exp(i sign 2 pi c s_q / 2^(j-m+1)) where c is the Hadamard's output
    bit (forward) or input bit (adjoint, carry_input=True), passed along a bond
    of size two through the sites between sites[m] and sites[-1]."""
    h, last = sites[m], sites[-1]
    later = {q: j - m for j, q in enumerate(sites) if j > m}
    out = []
    for n in range(L):
        if n < h or n > last or (h == last and n != h):
            out.append(_identity_site())
            continue
        if n == h:
            bond = 2 if h < last else 1
            t = np.zeros((1, 2, 2, bond), dtype=np.complex128)
            for u in range(2):
                for s in range(2):
                    c = (s if carry_input else u) if bond == 2 else 0
                    t[0, u, s, c] = -_R2 if (u and s) else _R2
            out.append(t)
            continue
        bond = 2 if n < last else 1
        t = np.zeros((2, 2, 2, bond), dtype=np.complex128)
        rel = later.get(n)
        for c in range(2):
            for s in range(2):
                w = 1.0 if rel is None else np.exp(1j * sign * 2.0 * np.pi * c * s / 2.0 ** (rel + 1))
                t[c, s, s, c if bond == 2 else 0] = w
        out.append(t)
    return out


def qft_mpo(n: int, inverse: bool = False, sites: Optional[Sequence[int]] = None) -> ttlab.MPOList:
    """qft.hpp:67-101: the layers in matrix order (last factor acts first)."""
    if n < 1:
        raise ttlab.ShapeError("qft_mpo: need at least one site")
    if sites is None:
        subset = list(range(n))
    else:
        subset = [int(q) for q in sites]
        if not subset:
            raise ttlab.ShapeError("qft_mpo: empty site subset")
        if any(a >= b for a, b in zip(subset[:-1], subset[1:])):
            raise ttlab.ShapeError("qft_mpo: sites must be strictly ascending")
        if subset[0] < 0 or subset[-1] >= n:
            raise ttlab.ShapeError("qft_mpo: site subset out of range")
    sign = 1.0 if inverse else -1.0
    order = range(len(subset)) if inverse else range(len(subset) - 1, -1, -1)
    return ttlab.MPOList([qft_layer(n, subset, m, sign, inverse) for m in order])


def iqft_mpo(n: int, sites: Optional[Sequence[int]] = None) -> ttlab.MPOList:
    return qft_mpo(n, True, sites)


def _length(v) -> int:
    return len(v) if not isinstance(v, ttlab.DeviceMPS) else v.info()["n"]


def qft(v, strategy: ttlab.Strategy = ttlab.DEFAULT_STRATEGY) -> ttlab.DeviceMPS:
    """qft.hpp:107-109."""
    return ttlab.apply(qft_mpo(_length(v)), v, strategy)


def iqft(v, strategy: ttlab.Strategy = ttlab.DEFAULT_STRATEGY) -> ttlab.DeviceMPS:
    """qft.hpp:110-112."""
    return ttlab.apply(qft_mpo(_length(v), True), v, strategy)


def qft_flip(v):
    """qft.hpp:116-126: reversed site order with transposed bonds (bit reversal
    of the dense index).  Host tensors in, host tensors out; a DeviceMPS is
    read back and re-uploaded with its error bound."""
    if isinstance(v, ttlab.DeviceMPS):
        ts = [np.ascontiguousarray(t.transpose(2, 1, 0)) for t in reversed(v.to_tensors())]
        return ttlab.DeviceMPS.from_tensors(ts, error=v.error(), ctx=v.ctx)
    return [np.ascontiguousarray(np.asarray(t).transpose(2, 1, 0)) for t in reversed(list(v))]
