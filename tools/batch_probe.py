"""Batched simplify beyond the C5 shapes: more than 16 chains (no grid kernels) with splits too large for the
shared-memory panel, so the one-CTA Jacobi works from the planned global workspace.  Every 5th chain is compared
with the oracle."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import ttlab_oracle as O  # noqa: E402
from paper_2601_16734_b200 import inputs as I  # noqa: E402
from paper_2601_16734_b200 import ttlab  # noqa: E402
from tests._compare import distance  # noqa: E402

nb, n, chi, out = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (20, 10, 96, 48)))
chains = [I.random_mps(n, 2, chi, 900 + i) for i in range(nb)]
strat = dict(max_bond=out, max_sweeps=2)
t0 = time.time()
rep = []
g = ttlab.simplify(ttlab.DeviceMPS.from_batch(chains), ttlab.Strategy(**strat), report=rep)
print("gpu %.2f s for %d chains" % (time.time() - t0, nb))
worst = 0.0
for i in range(0, nb, 5):
    rr = {}
    ref = O.simplify(O.MPS(chains[i]), O.Strategy(**strat), fast=True, report=rr)
    ts = g.to_tensors(i)
    assert g.bond_dimensions(i) == ref.bond_dimensions(), (i, g.bond_dimensions(i), ref.bond_dimensions())
    d = distance(ts, ref.tensors) / ref.norm()
    worst = max(worst, d)
    print(i, "distance %.2e" % d, "sweeps", rep[i]["sweeps"], rr["sweeps"], "residual", rep[i]["residual"], rr["residual"])
    assert d <= 1e-10 and rep[i]["sweeps"] == rr["sweeps"] and abs(rep[i]["residual"] - rr["residual"]) <= 1e-10 * max(1.0, ref.norm()), (i, d)
print("OK, worst distance %.2e" % worst)
