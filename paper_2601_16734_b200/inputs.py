"""Seeded synthetic inputs for the five BASELINE configs.

The reference publishes no dataset; BASELINE.json defines the inputs
(i.i.d. N(0,1) entries, bond profile min(chi, d^k, d^(n-k)) as in
`random_uniform_mps`, mps.hpp:500-506, normalised to unit norm with
`MPS::scaled` semantics, mps.hpp:98-117).  The generator is counter based so
any element can be regenerated independently of the others:

    key(seed, chain, site) = splitmix64 chain over the three integers
    u_k = (splitmix64(key + 2e + k) >> 11 + 0.5) * 2^-53,  k = 0, 1
    x_e = sqrt(-2 ln u_0) * cos(2 pi u_1)           (Box-Muller)

Complex tensors draw the real part at element 2e and the imaginary part at 2e+1
of the same counter stream.  Both the GPU run and the CPU oracle consume the
exact same arrays.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _key(*ints: int) -> np.uint64:
    k = np.uint64(0x243F6A8885A308D3)
    for v in ints:
        k = _splitmix64(np.asarray(k ^ np.uint64(v & 0xFFFFFFFFFFFFFFFF), dtype=np.uint64))
    return np.uint64(k)


def normals(count: int, seed: int, chain: int, site: int) -> np.ndarray:
    """`count` i.i.d. N(0,1) doubles for tensor (seed, chain, site)."""
    key = _key(seed, chain, site)
    e = np.arange(count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        c0 = key + np.uint64(2) * e
    u0 = ((_splitmix64(c0) >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
    u1 = ((_splitmix64(c0 + np.uint64(1)) >> np.uint64(11)).astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)
    return np.sqrt(-2.0 * np.log(u0)) * np.cos(2.0 * math.pi * u1)


def bond_profile(n: int, d: int, chi: int) -> List[int]:
    """min(chi, d^k, d^(n-k)) for k = 0..n (mps.hpp:500-506)."""
    out = []
    for k in range(n + 1):
        cap = min(float(chi), float(d) ** k, float(d) ** (n - k))
        out.append(int(max(1.0, cap)))
    return out


def _norm2(tensors) -> float:
    env = np.ones((1, 1), dtype=tensors[0].dtype)
    for t in tensors:
        x = np.tensordot(env, t, axes=([1], [0]))
        env = np.tensordot(t.conj(), x, axes=([0, 1], [0, 1]))
    return float(np.real(env[0, 0]))


def scale_to_unit(tensors):
    """MPS::scaled(1/|psi|) semantics: |f|^(1/n) on every site (mps.hpp:98-117)."""
    nrm = math.sqrt(max(0.0, _norm2(tensors)))
    root = (1.0 / nrm) ** (1.0 / len(tensors))
    return [t * root for t in tensors]


def random_mps(n: int, d: int, chi: int, seed: int, chain: int = 0, complex_: bool = False,
               normalise: bool = True) -> List[np.ndarray]:
    bonds = bond_profile(n, d, chi)
    ts = []
    for k in range(n):
        shape = (bonds[k], d, bonds[k + 1])
        cnt = int(np.prod(shape))
        if complex_:
            z = normals(2 * cnt, seed, chain, k)
            ts.append((z[0::2] + 1j * z[1::2]).reshape(shape))
        else:
            ts.append(normals(cnt, seed, chain, k).reshape(shape))
    return scale_to_unit(ts) if normalise else ts


def laplacian_mpo(n: int) -> List[np.ndarray]:
    """Periodic QTT second difference D_{+1} + D_{-1} - 2 I on 2^n points,
    bond D = 3, entries in {-2, 1, 0}.  B[c, j(out), i(in), c']."""
    I = np.eye(2)
    E01 = np.array([[0.0, 1.0], [0.0, 0.0]])
    E10 = np.array([[0.0, 0.0], [1.0, 0.0]])
    Z = np.zeros((2, 2))
    W = [[I, E01, E10], [Z, E10, Z], [Z, Z, E01]]  # rows = left bond, cols = right bond

    def tensor(blocks):  # blocks[c][c'] -> B[c, j, i, c']
        L, R = len(blocks), len(blocks[0])
        t = np.zeros((L, 2, 2, R))
        for c in range(L):
            for cp in range(R):
                t[c, :, :, cp] = blocks[c][cp]
        return t

    first = [[W[0][cp] + W[1][cp] + W[2][cp] for cp in range(3)]]  # [1,1,1] W
    vec = [-2.0, 1.0, 1.0]
    last = [[sum(W[c][cp] * vec[cp] for cp in range(3))] for c in range(3)]  # W [-2,1,1]^T
    return [tensor(first)] + [tensor(W) for _ in range(n - 2)] + [tensor(last)]


def random_mpo(n: int, d: int, D: int, seed: int) -> List[np.ndarray]:
    """Config 4 MPO: bonds min(D, (d^2)^k, (d^2)^(n-k)), entries N(0, 1/(D d))."""
    bonds = bond_profile(n, d * d, D)
    sd = 1.0 / math.sqrt(D * d)
    ts = []
    for k in range(n):
        shape = (bonds[k], d, d, bonds[k + 1])
        ts.append(sd * normals(int(np.prod(shape)), seed, 0, k).reshape(shape))
    return ts


@dataclass(frozen=True)
class Config:
    name: str
    kind: str  # "simplify" | "apply" | "hadamard" | "batch"
    n: int
    d: int
    chi: int
    out_chi: int
    tolerance: float
    max_sweeps: int
    complex_: bool = False
    mpo_D: int = 0
    batch: int = 1
    seed: int = 0


# SURVEY.md §8a/§8d, BASELINE.json "configs" (seeds per §8d)
CONFIGS = {
    "C1": Config("C1", "simplify", 20, 2, 32, 16, 1e-12, 4, seed=101),
    "C2": Config("C2", "apply", 20, 2, 64, 64, 1e-12, 4, mpo_D=3, seed=202),
    "C3": Config("C3", "hadamard", 24, 2, 64, 128, 1e-10, 4, complex_=True, seed=303),
    "C4": Config("C4", "apply", 30, 2, 512, 512, 1e-12, 2, mpo_D=8, seed=405),
    "C5": Config("C5", "batch", 20, 2, 128, 64, 1e-12, 4, batch=1024, seed=500),
}


def config_inputs(cfg: Config, chain: int = 0) -> Tuple[list, list]:
    """(target-side operands) for one chain: returns (mps_list, mpo) where the
    target is mps_list[0] (simplify/batch), apply_raw(mpo, mps_list[0]) or
    hadamard(mps_list[0], mps_list[1])."""
    if cfg.kind in ("simplify", "batch"):
        seed = cfg.seed + chain if cfg.kind == "batch" else cfg.seed
        return [random_mps(cfg.n, cfg.d, cfg.chi, seed)], None
    if cfg.kind == "apply":
        psi = random_mps(cfg.n, cfg.d, cfg.chi, cfg.seed)
        mpo = laplacian_mpo(cfg.n) if cfg.mpo_D == 3 else random_mpo(cfg.n, cfg.d, cfg.mpo_D, cfg.seed + 1)
        return [psi], mpo
    if cfg.kind == "hadamard":
        a = random_mps(cfg.n, cfg.d, cfg.chi, cfg.seed, complex_=True)
        b = random_mps(cfg.n, cfg.d, cfg.chi, cfg.seed + 1, complex_=True)
        return [a, b], None
    raise ValueError(cfg.kind)


def _batch_chain(args):
    name, chain = args
    return config_inputs(CONFIGS[name], chain=chain)[0][0]


def batch_inputs(cfg: Config, lo: int, hi: int, workers: int = 0) -> list:
    """Chains [lo, hi) of a batched config, generated on a pool of host processes
    (the counter-based generator makes every chain independent of the others)."""
    import multiprocessing as mp
    import os
    idx = list(range(lo, hi))
    workers = workers or min(len(idx), os.cpu_count() or 1)
    if workers <= 1 or len(idx) < 8:
        return [config_inputs(cfg, chain=c)[0][0] for c in idx]
    saved = {k: os.environ.get(k) for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS")}
    for k in saved:
        os.environ[k] = "1"  # single-threaded BLAS in the workers (inherited by the spawned processes)
    try:
        with mp.get_context("spawn").Pool(workers) as pool:
            return pool.map(_batch_chain, [(cfg.name, c) for c in idx], chunksize=max(1, len(idx) // (4 * workers)))
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
