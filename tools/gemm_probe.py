"""DMMA GEMM throughput on C4/C3-shaped contractions (device buffers, kernel time only)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2601_16734_b200._lib import lib  # noqa: E402

SHAPES = [  # (name, opA, opB, M, N, K)
    ("C4 X=L*T_n", 0, 0, 512, 8192, 4096),
    ("C4 Y=X*T_n+1", 0, 0, 1024, 8192, 4096),
    ("C4 theta=Y*R^T", 0, 1, 2048, 512, 4096),
    ("C4 env=psi^H*X", 2, 0, 512, 4096, 1024),
    ("C4 QR carry R*T", 0, 0, 4096, 8192, 4096),
    ("square 4096", 0, 0, 4096, 4096, 4096),
    ("C2 Y", 0, 0, 128, 384, 192),
]
ONLY = sys.argv[1] if len(sys.argv) > 1 else None
for cplx in (False, True):
    for name, oa, ob, M, N, K in SHAPES:
        if ONLY and (ONLY not in name or cplx):
            continue
        dt = torch.complex128 if cplx else torch.float64
        A = torch.randn(M * K, dtype=dt, device="cuda")
        B = torch.randn(K * N, dtype=dt, device="cuda")
        Cm = torch.empty(M * N, dtype=dt, device="cuda")
        ms = C.c_double()
        reps = 3 if M * N * K > 1e9 else 20
        st = lib.ttg_debug_gemm_dev(1 if cplx else 0, oa, ob, M, N, K, 1, C.c_void_p(A.data_ptr()),
                                    C.c_void_p(B.data_ptr()), C.c_void_p(Cm.data_ptr()), reps, C.byref(ms))
        fl = (8 if cplx else 2) * M * N * K
        print(f"{'c128' if cplx else 'f64 '} {name:18s} {M}x{N}x{K}: st={st} {ms.value * 1e3:9.1f} us "
              f"{fl / ms.value / 1e9:7.2f} TF/s ({100 * fl / ms.value / 1e9 / 37.07:5.1f}% of DMMA peak)", flush=True)
