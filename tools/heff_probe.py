"""Two-site H_eff matvec (eigensolvers.hpp:15-64) at C4-like sizes: device call through the C-ABI
(host buffers, H2D/D2H included) vs the oracle restatement on the host.
Usage: python tools/heff_probe.py [chi] [D]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import ttlab_oracle as O  # noqa: E402  (checker / CPU leg only)
from paper_2601_16734_b200 import ttlab as t  # noqa: E402

chi = int(sys.argv[1]) if len(sys.argv) > 1 else 512
D = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rng = np.random.default_rng(1)
L = rng.standard_normal((D, chi, chi))
R = rng.standard_normal((D, chi, chi))
w1 = rng.standard_normal((D, 2, 2, D)) / np.sqrt(2 * D)
w2 = rng.standard_normal((D, 2, 2, D)) / np.sqrt(2 * D)
x = rng.standard_normal(chi * 4 * chi)
y = t.apply_effective_two_site(L, w1, w2, R, x)  # warm-up (context, allocations)
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    y = t.apply_effective_two_site(L, w1, w2, R, x)
gpu_ms = (time.perf_counter() - t0) / reps * 1e3
t0 = time.perf_counter()
ref = O.apply_effective_two_site(L, w1, w2, R, x)
cpu_ms = (time.perf_counter() - t0) * 1e3
err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
flops = 2 * D * chi * chi * 4 * chi * 2  # the two GEMM stages
print(f"chi={chi} D={D}: device call {gpu_ms:.2f} ms (host buffers, {flops / 1e9:.1f} GF in the GEMMs), "
      f"oracle {cpu_ms:.0f} ms, rel.err {err:.1e}")
