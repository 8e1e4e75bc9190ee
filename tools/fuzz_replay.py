"""Replay the splits of a failing fuzz case (gpurun_out/fuzz_fail_*.pkl) one by one: the oracle's simplify is
run with a hook recording every schmidt_split input; each is then given to the device split
(ttg_schmidt_split) with the same strategy, and rank / dropped weight / reconstruction are compared."""
import pickle
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import ttlab_oracle as O  # noqa: E402
from paper_2601_16734_b200 import ttlab as t  # noqa: E402

d = pickle.load(open(sys.argv[1], "rb"))
desc = d["desc"]
print(desc)
kw = dict(method=desc["method"], tolerance=desc["tolerance"], max_sweeps=desc["max_sweeps"], normalize=desc["normalize"])
so = O.Strategy(max_bond=desc["max_bond"] or O.UNBOUNDED_BOND, **kw)
sg = t.Strategy(max_bond=desc["max_bond"] or t.UNBOUNDED_BOND, **kw)
calls = []
orig = O.schmidt_split


def hook(theta, strategy, direction=O.LEFT_TO_RIGHT):
    out = orig(theta, strategy, direction)
    calls.append((np.array(theta), strategy, direction, out))
    return out


O.schmidt_split = hook
om = lambda ts: O.MPS([np.asarray(x) for x in ts], 0.0)  # noqa: E731
if desc["op"] == "simplify":
    O.simplify(om(d["a"]), so)
elif desc["op"] == "hadamard":
    O.simplify(O.hadamard(om(d["a"]), om(d["b"])), so)
else:
    O.simplify_sum(O.MPSSum(desc["weights"], [om(s) for s in d["states"]]), so)
O.schmidt_split = orig
print(len(calls), "splits")
for i, (theta, strat, direction, (a, b, err)) in enumerate(calls):
    gs = t.Strategy(method=strat.method, tolerance=strat.tolerance,
                    simplification_tolerance=strat.simplification_tolerance,
                    max_bond=strat.max_bond if strat.max_bond < (1 << 40) else t.UNBOUNDED_BOND,
                    max_sweeps=strat.max_sweeps, normalize=strat.normalize)
    ga, gb, gerr = t.schmidt_split(theta, gs, direction)
    rec = np.linalg.norm(ga @ gb - a @ b) / max(np.linalg.norm(a @ b), 1e-300)
    ok = ga.shape == a.shape and rec < 1e-9 and abs(gerr - err) <= 1e-10 * max(np.linalg.norm(theta), 1e-300)
    print(f"{'ok ' if ok else 'BAD'} split {i}: theta {theta.shape} {theta.dtype} dir {direction} tol {strat.tolerance:g} "
          f"rank ref {a.shape[1]} gpu {ga.shape[1]} err ref {err:.3e} gpu {gerr:.3e} rec {rec:.2e}")
    if not ok:
        np.save(f"gpurun_out/bad_theta_{i}.npy", theta)
