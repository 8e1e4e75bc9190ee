"""One call of a config (for ncu launch lists)."""
import sys

sys.path.insert(0, ".")
from paper_2601_16734_b200 import inputs as I  # noqa: E402
from paper_2601_16734_b200 import ttlab  # noqa: E402

cfg = I.CONFIGS[sys.argv[1]]
mps, W = I.config_inputs(cfg)
strat = ttlab.Strategy(max_bond=cfg.out_chi, tolerance=cfg.tolerance, max_sweeps=cfg.max_sweeps)
if cfg.kind == "apply":
    out = ttlab.apply(W, mps[0], strat)
elif cfg.kind == "hadamard":
    out = ttlab.simplify(ttlab.hadamard(mps[0], mps[1]), strat)
else:
    out = ttlab.simplify(mps[0], strat)
print("bonds", out.bond_dimensions())
