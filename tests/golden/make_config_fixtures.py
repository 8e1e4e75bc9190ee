"""Oracle fixtures for the full-size configs whose CPU run takes minutes (C3, C4).

TEST INFRASTRUCTURE.  Usage (from the repo root, in the build container):

    python tests/golden/make_config_fixtures.py C4 [C3 ...]

Runs the oracle restatement (oracle/ttlab_oracle.py, native dtype, minimal
contraction order: same values as the reference's pair-first order) on the
exact seeded inputs the GPU tests use (paper_2601_16734_b200/inputs.py) and
writes

  tests/golden/<cfg>_oracle.json   (committed) the gauge-invariant results of
      SURVEY.md §8c: output bond dims, per-bond Schmidt spectra of the final
      output from an exact canonical pass, residual, <T,T>, |psi|, <psi, T>,
      sweeps and the dist^2 history, plus the relative Schmidt gap
      (s_{r-1} - s_r) / s_{r-1} at every truncating split;
  tests/golden/<cfg>_psi_ref.npz   (git-ignored, 6-56 MB) the oracle's output
      tensors for the cancellation-free distance |psi_gpu - psi_ref| (metric 6).
      The file travels to the GPU box with the working tree (gpurun snapshot).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ttlab_oracle as O  # noqa: E402
from paper_2601_16734_b200 import inputs as I  # noqa: E402
from tests._compare import spectra  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def run(name):
    cfg = I.CONFIGS[name]
    mps, W = I.config_inputs(cfg)
    strat = O.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
    if cfg.kind == "apply":
        target = O.apply_raw(O.MPO(W), O.MPS(mps[0]))
    elif cfg.kind == "hadamard":
        target = O.hadamard(O.MPS(mps[0]), O.MPS(mps[1]))
    else:
        target = O.MPS(mps[0])
    O.GAP_LOG = []
    t0 = time.time()
    rep = {}
    psi = O.simplify(target, strat, fast=True, report=rep)
    t_run = time.time() - t0
    gaps = O.GAP_LOG
    O.GAP_LOG = None
    spec = spectra(psi.tensors)
    ov = O.scprod(psi, target)
    out = {
        "config": name, "strategy": {"max_bond": cfg.out_chi, "tolerance": cfg.tolerance,
                                     "max_sweeps": cfg.max_sweeps},
        "generator": "tests/golden/make_config_fixtures.py (oracle fast=True, native dtype)",
        "oracle_seconds": t_run,
        "bonds": psi.bond_dimensions(), "sweeps": rep["sweeps"], "residual": float(rep["residual"]),
        "target_norm2": float(rep["target_norm2"]), "dist2": [float(x) for x in rep["dist2"]],
        "error": float(psi.error), "norm": float(psi.norm()),
        "overlap": [float(np.real(ov)), float(np.imag(ov))],
        "spectra": [s.tolist() for s in spec],
        "min_rel_gap": min((g[5] for g in gaps), default=None),
        "gaps": gaps,
    }
    with open(os.path.join(HERE, f"{name}_oracle.json"), "w") as f:
        json.dump(out, f)
    np.savez(os.path.join(HERE, f"{name}_psi_ref.npz"), *psi.tensors)
    print(name, f"{t_run:.0f} s", "sweeps", rep["sweeps"], "residual", rep["residual"], "min gap", out["min_rel_gap"],
          flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        run(n)
