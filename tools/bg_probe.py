"""Block-Gram Jacobi (jacobi_bg.cu) vs the warp-pair grid kernel on C4-like real splits.
Usage: TTG_SVD_BG=<0|16|32> TTG_DEBUG_SVD_GRID=1 python tools/bg_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from wp_probe import c4_like, run  # noqa: E402

if __name__ == "__main__":
    tag = os.environ.get("TTG_SVD_BG", "default")
    for (m, n) in [(1024, 1024), (1024, 512), (512, 512), (600, 520), (256, 256)]:
        A = c4_like(m, n)
        L = np.ascontiguousarray(np.linalg.qr(A.T)[1].T)  # single R-only QR preconditioner: L = R^H
        run(L, 0)
        for mode in (0, 1):
            st, sw, ms, err, orth = run(L if mode == 0 else np.ascontiguousarray(L.T), mode)
            print(f"BG={tag} {m}x{n} f64 mode={mode}: st={st} sweeps={sw} {ms:8.2f} ms "
                  f"({ms / max(sw, 1):.3f} ms/sweep)  |ds|/s0={err:.1e} orth={orth:.1e}", flush=True)
