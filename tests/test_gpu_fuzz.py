"""Fixed-seed slices of the randomised sweeps (tools/fuzz_parity.py, fuzz_split.py, fuzz_scalars.py): random
ops, chain lengths, mixed physical dimensions, bonds, dtypes and strategies against the oracle / numpy.  The
long campaigns (tens of thousands of cases, NaN-poisoned workspaces) are run by hand; these slices keep the
tools and the classes of input that found the two bugs of round 2 in the suite."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tool,args", [("fuzz_parity.py", ["300", "1"]), ("fuzz_parity.py", ["40", "4", "big"]),
                                       ("fuzz_split.py", ["500", "1"]), ("fuzz_scalars.py", ["300", "1"])])
def test_randomised_sweep(tool, args):
    r = subprocess.run([sys.executable, os.path.join("tools", tool)] + args, cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    tail = "\n".join(r.stdout.strip().splitlines()[-15:])
    assert r.returncode == 0, tail + r.stderr[-2000:]
    assert "FAIL" not in r.stdout, tail
