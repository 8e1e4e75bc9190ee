"""Restatement of the reference's random inputs (TEST INFRASTRUCTURE ONLY).

`random_uniform_mps` (ref: proj/include/ttlab/mps.hpp:493-514) and the test
helper `oracle::random_matrix` (ref: proj/tests/test_utils.hpp:31-39) draw
`cplx(dist(rng), dist(rng))` from `std::mt19937_64` and
`std::uniform_real_distribution<double>(-1, 1)`.  libstdc++ maps one 64-bit
draw x to `double(x) / 2**64` (generate_canonical with k = 1), then to
`u * (b - a) + a`.  Pinned bit-for-bit against tests/golden/mt19937_64_uniform.json
(dumped by oracle/golden_rng.cpp under g++/libstdc++).
"""
from __future__ import annotations

import numpy as np

_N, _M = 312, 156
_MATRIX_A = 0xB5026F5AA96619E9
_UPPER = 0xFFFFFFFF80000000
_LOWER = 0x000000007FFFFFFF
_MASK = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (C++11 26.5.5 [rand.predef])."""

    def __init__(self, seed: int):
        mt = [0] * _N
        mt[0] = seed & _MASK
        for i in range(1, _N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _MASK
        self._mt = np.array(mt, dtype=np.uint64)
        self._buf = np.empty(0, dtype=np.uint64)
        self._pos = 0

    def _twist(self) -> np.ndarray:
        mt = self._mt
        u64 = np.uint64
        # the recurrence is sequential in blocks of _M; do it in three vector steps
        for lo, hi in ((0, _N - _M), (_N - _M, _N - 1)):
            y = (mt[lo:hi] & u64(_UPPER)) | (mt[lo + 1:hi + 1] & u64(_LOWER))
            mag = np.where((y & u64(1)) != 0, u64(_MATRIX_A), u64(0))
            src = np.arange(lo, hi) + _M
            src = np.where(src >= _N, src - _N, src)
            mt[lo:hi] = mt[src] ^ (y >> u64(1)) ^ mag
        y = (mt[_N - 1] & u64(_UPPER)) | (mt[0] & u64(_LOWER))
        mag = u64(_MATRIX_A) if int(y) & 1 else u64(0)
        mt[_N - 1] = mt[_M - 1] ^ (y >> u64(1)) ^ mag
        # tempering
        x = mt.copy()
        x ^= (x >> u64(29)) & u64(0x5555555555555555)
        x ^= (x << u64(17)) & u64(0x71D67FFFEDA60000)
        x ^= (x << u64(37)) & u64(0xFFF7EEE000000000)
        x ^= x >> u64(43)
        return x

    def draw(self, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        filled = 0
        while filled < count:
            if self._pos >= self._buf.size:
                self._buf = self._twist()
                self._pos = 0
            take = min(count - filled, self._buf.size - self._pos)
            out[filled:filled + take] = self._buf[self._pos:self._pos + take]
            self._pos += take
            filled += take
        return out


def _canonical(x: np.ndarray) -> np.ndarray:
    u = x.astype(np.float64) / 18446744073709551616.0
    return np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)


def uniform_pm1(rng: MT19937_64, count: int) -> np.ndarray:
    """`count` draws of uniform_real_distribution<double>(-1, 1)."""
    return _canonical(rng.draw(count)) * 2.0 + (-1.0)


def complex_draws(rng: MT19937_64, count: int) -> np.ndarray:
    """`count` values of cplx(dist(rng), dist(rng)).  g++ evaluates the two
    constructor arguments right to left, so the imaginary part is the first
    draw of each pair (pinned by tests/golden/mt19937_64_uniform.json)."""
    u = uniform_pm1(rng, 2 * count)
    return u[1::2] + 1j * u[0::2]


def random_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """ref: proj/tests/test_utils.hpp:31-39 (column-major fill)."""
    vals = complex_draws(MT19937_64(seed), rows * cols)
    return vals.reshape(cols, rows).T.copy()


def random_vector(n: int, seed: int) -> np.ndarray:
    """ref: proj/tests/test_utils.hpp:22-29."""
    return complex_draws(MT19937_64(seed), n)
