"""Randomised sweep over the device split (ttg_schmidt_split: every Jacobi / preconditioner kernel variant is
selected by shape): random m x n up to 320 (with a bias to odd and tiny sizes), real / complex, both directions,
random tolerance and max_bond, graded and rank-deficient spectra.  Checked against numpy's SVD: rank rule
(schmidt.hpp:40-59), dropped weight, |theta - a b| = dropped weight, isometry of the orthonormal factor.

    python tools/fuzz_split.py [cases] [seed] [big]      ("big": 200 .. 1600 rows / columns, the grid, cluster,
                                                          block-Gram and blocked-QR paths at odd sizes)"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2601_16734_b200 import ttlab as t  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 500
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
bad = 0
t0 = time.time()
BIG = len(sys.argv) > 3 and sys.argv[3] == "big"
for i in range(cases):
    big = rng.random() < 0.25
    m = int(rng.integers(1, 320 if big else 70))
    n = int(rng.integers(1, 320 if big else 70))
    cplx = rng.random() < 0.4
    if BIG:
        cplx = rng.random() < 0.3
        top = 1000 if cplx else 1600
        m, n = int(rng.integers(200, top)), int(rng.integers(200, top))
    kind = str(rng.choice(["gauss", "graded", "lowrank", "clustered"]))
    k = min(m, n)

    def rnd(*s):
        x = rng.standard_normal(s)
        return x + 1j * rng.standard_normal(s) if cplx else x

    if kind == "gauss":
        th = rnd(m, n)
    else:
        u, _ = np.linalg.qr(rnd(m, k))
        v, _ = np.linalg.qr(rnd(n, k))
        if kind == "graded":
            sv = 10.0 ** (-rng.uniform(0, 14) * np.arange(k) / max(k - 1, 1))
        elif kind == "lowrank":
            r = int(rng.integers(1, k + 1))
            sv = np.concatenate([rng.uniform(0.5, 2.0, r), np.zeros(k - r)])
        else:
            sv = np.sort(1.0 + 1e-9 * rng.standard_normal(k))[::-1]
        th = (u * sv) @ v.conj().T
    tol = float(rng.choice([0.0, 1e-12, 1e-8, 1e-3]))
    mb = int(rng.integers(1, k + 2)) if rng.random() < 0.5 else 0
    direction = int(rng.integers(0, 2))
    desc = dict(m=m, n=n, cplx=cplx, kind=kind, tol=tol, max_bond=mb, direction=direction)
    try:
        a, b, err = t.schmidt_split(th, t.Strategy(tolerance=tol, max_bond=mb or t.UNBOUNDED_BOND), direction)
    except Exception as e:  # noqa: BLE001
        bad += 1
        print(f"FAIL {i} {desc}: {type(e).__name__} {e}", flush=True)
        continue
    s = np.linalg.svd(th, compute_uv=False)
    nrm = max(np.linalg.norm(th), 1e-300)
    cutoff = tol * s[0]
    rank = max(1, int(np.sum(s > cutoff)))
    if mb:
        rank = min(rank, mb)
    r = a.shape[1]
    problems = []
    # a singular value within rounding of the cutoff (or of zero for tol = 0) may fall on either side
    near = np.abs(s - cutoff) <= 1e-10 * s[0] + 1e-13 * nrm
    lo = max(1, int(np.sum((s > cutoff) & ~near)))
    hi = max(1, int(np.sum((s > cutoff) | near)))
    if mb:
        lo, hi = min(lo, mb), min(hi, mb)
    if not lo <= r <= hi:
        problems.append(f"rank {r} not in [{lo}, {hi}] (numpy rule {rank})")
    else:
        want = np.sqrt(np.sum(s[r:] ** 2))
        if abs(err - want) > 1e-10 * nrm:
            problems.append(f"dropped weight {err:.6e} != {want:.6e}")
        res = np.linalg.norm(th - a @ b)
        if abs(res - want) > 1e-10 * nrm:
            problems.append(f"|theta - a b| {res:.6e} != dropped weight {want:.6e}")
        iso = a if direction == 0 else b.conj().T
        defect = np.abs(iso.conj().T @ iso - np.eye(r)).max()
        if defect > 1e-11:
            problems.append(f"isometry defect {defect:.2e}")
    if problems:
        bad += 1
        print(f"FAIL {i} {desc}: " + "; ".join(problems), flush=True)
print(f"{cases - bad} / {cases} splits agree ({time.time() - t0:.0f} s, seed {seed})")
sys.exit(1 if bad else 0)
