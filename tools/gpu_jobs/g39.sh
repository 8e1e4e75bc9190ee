set -u
python - <<'PY'
import os, sys
sys.argv = ["fuzz", "224", "2"]
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import numpy as np
import fuzz_parity as F
rng = np.random.default_rng(2)
for i in range(224):
    F.SKIP[0] = i < 222
    if i == 223:
        os.environ["TTG_DEBUG_SPLITS"] = "1"
    desc, problems = F.one_case(rng)
    if i >= 222:
        print(i, desc, problems, flush=True)
PY
