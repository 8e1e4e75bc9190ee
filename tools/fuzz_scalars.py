"""Randomised sweep over the scalar entry points and the centre moves: scprod, norm, expectation_mpo,
expectation_local (one- and two-point) and recenter with truncation, on chains with mixed physical dimensions,
unequal bra / ket bonds, real / complex operands; device path against the oracle.

    python tools/fuzz_scalars.py [cases] [seed]"""
import sys
import time

import numpy as np

sys.path.insert(0, "tools")
sys.path.insert(0, ".")
from fuzz_parity import rand_mpo, rand_mps  # noqa: E402
from oracle import ttlab_oracle as O  # noqa: E402
from paper_2601_16734_b200 import ttlab as t  # noqa: E402
from tests._compare import distance  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 500
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rng = np.random.default_rng(seed)
om = lambda ts: O.MPS([np.asarray(x) for x in ts], 0.0)  # noqa: E731
bad = 0
t0 = time.time()
for i in range(cases):
    op = str(rng.choice(["scprod", "norm", "expectation_mpo", "expectation_local", "recenter", "heff"]))
    n = int(rng.integers(1, 11))
    dims = [int(rng.choice([2, 2, 3, 4])) for _ in range(n)]
    cu, cv, cw = (bool(rng.random() < 0.4) for _ in range(3))
    u = rand_mps(rng, dims, int(rng.integers(1, 40)), cu)
    v = rand_mps(rng, dims, int(rng.integers(1, 40)), cv)
    desc = dict(op=op, dims=dims, cplx=(cu, cv, cw))
    problems = []
    try:
        if op == "scprod":
            got, ref = complex(t.scprod(u, v)[0]), complex(O.scprod(om(u), om(v)))
            sc = max(om(u).norm() * om(v).norm(), 1e-300)
            if abs(got - ref) > 1e-12 * sc:
                problems.append(f"{got} != {ref}")
        elif op == "norm":
            got, ref = float(t.norm(u)[0]), om(u).norm()
            if abs(got - ref) > 1e-12 * max(ref, 1e-300):
                problems.append(f"{got} != {ref}")
        elif op == "expectation_mpo":
            W = rand_mpo(rng, dims, int(rng.integers(1, 5)), cw)
            got = complex(t.expectation_mpo(W, u, v)[0])
            ref = complex(O.expectation_mpo(O.MPO(W), om(u), om(v)))
            sc = max(om(u).norm() * om(v).norm(), 1e-300) * 10.0
            if abs(got - ref) > 1e-11 * sc:
                problems.append(f"{got} != {ref}")
        elif op == "expectation_local":
            s1 = int(rng.integers(0, n))
            a = rng.standard_normal((dims[s1], dims[s1])) + (1j * rng.standard_normal((dims[s1], dims[s1])) if cw else 0)
            if n > 1 and rng.random() < 0.5:
                s2 = int(rng.choice([x for x in range(n) if x != s1]))
                b = rng.standard_normal((dims[s2], dims[s2])) + 0j
                got = complex(t.expectation_local(u, a, s1, b, s2)[0])
                ref = complex(O.expectation_local(om(u), a, s1, b, s2))
            else:
                got = complex(t.expectation_local(u, a, s1)[0])
                ref = complex(O.expectation_local(om(u), a, s1))
            sc = max(om(u).norm() ** 2, 1e-300) * 10.0
            if abs(got - ref) > 1e-11 * sc:
                problems.append(f"{got} != {ref}")
        elif op == "heff":  # y = H_eff x around a random pair, bra != ket (eigensolvers.hpp:15-64)
            if n < 2:
                continue
            W = rand_mpo(rng, dims, int(rng.integers(1, 5)), cw)
            k = int(rng.integers(0, n - 1))
            desc.update(site=k, D=int(np.asarray(W[k]).shape[3]))
            cp = lambda a: np.asarray(a, dtype=np.complex128)  # noqa: E731
            L = np.ones((1, 1, 1), dtype=np.complex128)
            for j in range(k):
                L = O.update_left_op_environment(L, cp(u[j]), cp(W[j]), cp(v[j]))
            R = np.ones((1, 1, 1), dtype=np.complex128)
            for j in range(n - 1, k + 1, -1):
                R = O.update_right_op_environment(R, cp(u[j]), cp(W[j]), cp(v[j]))
            x = np.einsum("asb,btc->astc", cp(v[k]), cp(v[k + 1])).reshape(-1)
            ref = O.apply_effective_two_site(L, cp(W[k]), cp(W[k + 1]), R, x)
            got = np.asarray(t.apply_effective_two_site(L, cp(W[k]), cp(W[k + 1]), R, x)).reshape(-1)
            if got.shape != ref.reshape(-1).shape or np.linalg.norm(got - ref.reshape(-1)) > 1e-11 * max(np.linalg.norm(ref), 1e-300):
                problems.append(f"|y - y_ref| {np.linalg.norm(got - ref.reshape(-1)):.2e} of {np.linalg.norm(ref):.2e}")
        else:  # canonicalize, then move the centre with truncation (mps.hpp:268-279)
            c0, c1 = int(rng.integers(0, n)), int(rng.integers(0, n))
            mb = int(rng.integers(1, 20))
            desc.update(c0=c0, c1=c1, max_bond=mb)
            so = O.Strategy(method=O.SVD_TRUNCATE, max_bond=mb)
            sg = t.Strategy(method=t.SVD_TRUNCATE, max_bond=mb)
            rc = O.canonicalize(om(u), c0, O.NO_TRUNCATION)
            rc.recenter(c1, so)
            gc = t.canonicalize(u, c0, t.NO_TRUNCATION)
            moved, err = t.recenter(gc, c1, sg)
            ts = moved.to_tensors()
            if [x.shape for x in ts] != [x.shape for x in rc.tensors]:
                problems.append("bonds differ")
            elif distance(ts, rc.tensors) > 1e-10 * max(rc.norm(), 1e-300):
                problems.append(f"distance {distance(ts, rc.tensors):.2e}")
    except Exception as e:  # noqa: BLE001
        problems.append(f"{type(e).__name__}: {e}")
    if problems:
        bad += 1
        print(f"FAIL {i} {desc}: " + "; ".join(problems), flush=True)
print(f"{cases - bad} / {cases} agree ({time.time() - t0:.0f} s, seed {seed})")
sys.exit(1 if bad else 0)
