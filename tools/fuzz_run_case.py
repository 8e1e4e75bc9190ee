"""Run one dumped fuzz case (tools/fuzz_cases/*.pkl) through the device path and print bonds / norm / error
next to the oracle's; with TTG_DEBUG_SPLITS=1 the library prints every split."""
import pickle
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import ttlab_oracle as O  # noqa: E402
from paper_2601_16734_b200 import ttlab as t  # noqa: E402
from tests._compare import distance  # noqa: E402

d = pickle.load(open(sys.argv[1], "rb"))
desc = d["desc"]
kw = dict(method=desc["method"], tolerance=desc["tolerance"], max_sweeps=desc["max_sweeps"], normalize=desc["normalize"])
so = O.Strategy(max_bond=desc["max_bond"] or O.UNBOUNDED_BOND, **kw)
sg = t.Strategy(max_bond=desc["max_bond"] or t.UNBOUNDED_BOND, **kw)
om = lambda ts: O.MPS([np.asarray(x) for x in ts], 0.0)  # noqa: E731
orig = O.schmidt_split


def hook(theta, strategy, direction=O.LEFT_TO_RIGHT):
    out = orig(theta, strategy, direction)
    print(f"oracle split dir {direction} theta {theta.shape} -> rank {out[0].shape[1]}", file=sys.stderr)
    return out


O.schmidt_split = hook
if desc["op"] == "simplify":
    ref = O.simplify(om(d["a"]), so)
    print("---- device", file=sys.stderr)
    got = t.simplify(d["a"], sg)
elif desc["op"] == "hadamard":
    ref = O.simplify(O.hadamard(om(d["a"]), om(d["b"])), so)
    print("---- device", file=sys.stderr)
    got = t.simplify(t.hadamard(d["a"], d["b"]), sg)
else:
    ref = O.simplify_sum(O.MPSSum(desc["weights"], [om(s) for s in d["states"]]), so)
    print("---- device", file=sys.stderr)
    got = t.simplify(t.MPSSum(desc["weights"], d["states"]), sg)
ts = got.to_tensors()
print("bonds gpu", [x.shape[2] for x in ts], "ref", [x.shape[2] for x in ref.tensors])
print("norm gpu", float(t.norm(got)[0]), "ref", ref.norm(), "error gpu", got.error(), "ref", ref.error)
if [x.shape for x in ts] == [x.shape for x in ref.tensors]:
    print("distance", distance(ts, ref.tensors))
