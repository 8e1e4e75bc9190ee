"""Reference outputs for tests/ref_cases.py, produced by the REFERENCE'S OWN CODE.

TEST INFRASTRUCTURE.  Usage (build container, where /root/reference exists):

    make -C oracle            # oracle/_ref/ttlab_ref: reference headers + Eigen stand-in
    python tests/golden/make_ref_fixtures.py [case ...]

Every case of tests/ref_cases.CASES is written as TTLAB1 files (the reference's own container,
serialize.hpp), run through oracle/_ref/ttlab_ref (ref_driver.cpp: ttlab::apply / simplify /
canonicalize / hadamard / scprod / expectation_mpo called unchanged) and the outputs are stored
in tests/golden/ref_outputs.npz: per case the JSON line of the run (error ledger, norm, bond
dimensions, sweeps, residual) and the output tensors (real part only when the imaginary part is
identically zero).  The reference cannot travel to the GPU box; this file does.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from tests import ref_cases as R  # noqa: E402


def main(names):
    if not R.have_ref():
        sys.exit("oracle/_ref/ttlab_ref missing: run `make -C oracle` where /root/reference exists")
    arrays, meta = {}, {}
    if os.path.exists(R.FIXTURE) and names:  # partial refresh
        for name, (m, ts) in R.load_fixture().items():
            meta[name] = m
            for k, t in enumerate(ts or []):
                arrays["%s/%d" % (name, k)] = t
    for name in (names or list(R.CASES)):
        t0 = time.time()
        m, ts = R.run_reference(name)
        m["seconds"] = round(time.time() - t0, 2)
        m["sites"] = None if ts is None else len(ts)
        for k in [k for k in arrays if k.startswith(name + "/")]:
            del arrays[k]
        for k, t in enumerate(ts or []):
            arrays["%s/%d" % (name, k)] = t.real.copy() if not np.any(t.imag) else t
        meta[name] = m
        print(name, json.dumps(m), flush=True)
    np.savez_compressed(R.FIXTURE, meta=np.array(json.dumps(meta, sort_keys=True)), **arrays)
    print("wrote", R.FIXTURE, os.path.getsize(R.FIXTURE), "bytes")


if __name__ == "__main__":
    main(sys.argv[1:])
