"""Run one BASELINE config end to end on the GPU and check size-independent
properties (isometries, norm/residual consistency).  Usage: run_config.py C4"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2601_16734_b200 import flops as F  # noqa: E402
from paper_2601_16734_b200 import inputs as I  # noqa: E402
from paper_2601_16734_b200 import ttlab  # noqa: E402

name = sys.argv[1]
cfg = I.CONFIGS[name]
t0 = time.time()
mps, W = I.config_inputs(cfg)
print(f"inputs {time.time() - t0:.1f} s", flush=True)
ctx = ttlab.context()
strat = ttlab.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
dev = [ttlab.DeviceMPS.from_tensors(m) for m in mps]
Wd = ttlab.DeviceMPO(W) if W is not None else None


def run(profile=False):
    if profile:
        ctx.profile_enable(True)
    ctx.synchronize()
    t = time.time()
    rep = []
    if cfg.kind == "apply":
        out = ttlab.apply(Wd, dev[0], strat, report=rep)
    elif cfg.kind == "hadamard":
        out = ttlab.simplify(ttlab.hadamard(dev[0], dev[1]), strat, report=rep)
    else:
        out = ttlab.simplify(dev[0], strat, report=rep)
    ctx.synchronize()
    dt = time.time() - t
    prof = ctx.profile_read() if profile else None
    if profile:
        ctx.profile_enable(False)
    return out, rep[0], dt, prof


out, rep, dt, _ = run()
print(f"first call {dt:.2f} s  report {rep}", flush=True)
out, rep, dt, _ = run()
print(f"second call {dt:.2f} s", flush=True)
_, _, dtp, prof = run(profile=True)
ts = out.to_tensors()
bonds = out.bond_dimensions()
iso = 0.0
for A in ts[1:]:
    b = A.reshape(A.shape[0], -1)
    iso = max(iso, np.abs(b @ b.conj().T - np.eye(b.shape[0])).max())
nrm2 = float(np.vdot(ts[0], ts[0]).real)
dist = rep["residual"] - 32 * 2.220446049250313e-16 * np.sqrt(rep["target_norm2"])
consist = abs(rep["target_norm2"] - nrm2 - dist ** 2)
if cfg.kind == "apply":
    tb = [1] + [w.shape[3] * a.shape[2] for w, a in zip(W, mps[0])]
elif cfg.kind == "hadamard":
    tb = [1] + [a.shape[2] * b.shape[2] for a, b in zip(mps[0], mps[1])]
else:
    tb = [1] + [a.shape[2] for a in mps[0]]
fl = F.algorithmic_flops(tb, bonds, [2] * cfg.n, rep["sweeps"], complex_=cfg.complex_)
res = {"config": name, "seconds": dt, "sweeps": rep["sweeps"], "sweeps_per_s": rep["sweeps"] / dt,
       "F_alg_tflop": fl["F_alg"] / 1e12, "fp64_tflops_effective": fl["F_alg"] / dt / 1e12,
       "max_bond": max(bonds), "isometry_err": iso, "norm_consistency": consist, "report": rep, "profile": prof,
       "profiled_call_s": dtp}
print(json.dumps(res), flush=True)
