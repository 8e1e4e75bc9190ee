"""Beyond-config sizes: splits larger than the block-Gram kernel's 1024-row limit (theta up to 2048 x 2048)
and a non-power-of-two output bond, GPU vs oracle (fast=True) on the gauge-invariant results."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import ttlab_oracle as O  # noqa: E402
from paper_2601_16734_b200 import inputs as I  # noqa: E402
from paper_2601_16734_b200 import ttlab  # noqa: E402
from tests._compare import distance  # noqa: E402

n, chi, out = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (22, 1024, 768)))
cplx = len(sys.argv) > 4 and sys.argv[4] == "c"  # complex128 chain (splits beyond 512 rows: warp-pair kernel, E = 32)
psi = I.random_mps(n, 2, chi, 777, complex_=cplx)
strat = dict(max_bond=out, max_sweeps=1)
rep = []
t0 = time.time()
g = ttlab.simplify(psi, ttlab.Strategy(**strat), report=rep)
ts = g.to_tensors()
t1 = time.time()
rr = {}
ref = O.simplify(O.MPS(psi), O.Strategy(**strat), fast=True, report=rr)
t2 = time.time()
print("gpu %.2fs oracle %.2fs" % (t1 - t0, t2 - t1))
print("bonds equal", g.bond_dimensions() == ref.bond_dimensions(), max(g.bond_dimensions()))
print("sweeps", rep[0]["sweeps"], rr["sweeps"], "residual", rep[0]["residual"], rr["residual"])
d = distance(ts, ref.tensors) / ref.norm()
print("distance/|psi| %.3e" % d)
k = n // 2
a = ts[k + 1].reshape(ts[k + 1].shape[0], -1)
print("right-isometry err %.2e" % np.abs(a @ a.conj().T - np.eye(a.shape[0])).max())
assert g.bond_dimensions() == ref.bond_dimensions() and d <= 1e-10 and abs(rep[0]["residual"] - rr["residual"]) <= 1e-10
print("OK")
