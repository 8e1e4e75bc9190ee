import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import os
os.chdir(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
sys.path.insert(0, os.getcwd())
from tests.test_gpu_kernels import _svd
worst = 0.0
for n in (64, 128, 256):
    for seed in range(n, n + 8):
        rng = np.random.default_rng(seed)
        U, _ = np.linalg.qr(rng.standard_normal((n, n)))
        V, _ = np.linalg.qr(rng.standard_normal((n, n)))
        s = np.repeat([1.0, 0.5, 0.1, 1e-3], n // 4) * (1 + 1e-9 * rng.standard_normal(n))
        th = (U * s) @ V.T
        out = []
        for mode in (0, 1):
            iso, sv, r, _ = _svd(th, mode, tol=1e-12)
            e = np.abs(iso.conj().T @ iso - np.eye(r)).max() if mode == 0 else np.abs(iso @ iso.conj().T - np.eye(r)).max()
            out.append(e)
        print(n, seed, ["%.2e" % e for e in out], flush=True)
        worst = max(worst, max(out))


print("WORST %.3e" % worst)
