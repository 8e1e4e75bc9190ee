"""ctypes binding of the in-tree C-ABI library `libttgpu.so` (include/ttgpu.h).

There is no fallback: if the library is missing or cannot be loaded the import
fails loudly, and if no CUDA device is present every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TTG_LIB", os.path.join(_HERE, "libttgpu.so"))  # TTG_LIB: A/B builds (tools)

TTG_OK, TTG_SHAPE, TTG_CAPACITY, TTG_NUMERIC, TTG_CUDA, TTG_INVALID = range(6)
TTG_F64, TTG_C128 = 0, 1
TTG_SVD_TRUNCATE, TTG_VARIATIONAL = 0, 1


class ttg_strategy(C.Structure):
    _fields_ = [("method", C.c_int), ("tolerance", C.c_double), ("simplification_tolerance", C.c_double),
                ("max_bond", C.c_int64), ("max_sweeps", C.c_int), ("normalize", C.c_int)]


class ttg_report(C.Structure):
    _fields_ = [("sweeps", C.c_int), ("converged", C.c_int), ("residual", C.c_double), ("error", C.c_double),
                ("norm", C.c_double), ("target_norm2", C.c_double)]


class ttg_mps_view(C.Structure):
    _fields_ = [("n", C.c_int), ("dtype", C.c_int), ("bonds", C.POINTER(C.c_int64)),
                ("phys", C.POINTER(C.c_int64)), ("sites", C.POINTER(C.c_void_p)), ("error", C.c_double)]


class ttg_mpo_view(C.Structure):
    _fields_ = [("n", C.c_int), ("dtype", C.c_int), ("bonds", C.POINTER(C.c_int64)),
                ("phys_out", C.POINTER(C.c_int64)), ("phys_in", C.POINTER(C.c_int64)),
                ("sites", C.POINTER(C.c_void_p))]


# exported symbol -> (restype, argtypes); tests check this list against include/ttgpu.h
SIGNATURES = {
    "ttg_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "ttg_destroy": (None, [C.c_void_p]),
    "ttg_last_error": (C.c_char_p, [C.c_void_p]),
    "ttg_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ttg_synchronize": (C.c_int, [C.c_void_p]),
    "ttg_kernel_launches": (C.c_int64, [C.c_void_p]),
    "ttg_comm_unique_id": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ttg_comm_init": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "ttg_comm_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ttg_comm_allgather_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "ttg_comm_free": (C.c_int, [C.c_void_p]),
    "ttg_version": (C.c_char_p, []),
    "ttg_profile_enable": (C.c_int, [C.c_void_p, C.c_int]),
    "ttg_profile_svd_sweeps": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "ttg_profile_read": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double)]),
    "ttg_mps_upload": (C.c_int, [C.c_void_p, C.POINTER(ttg_mps_view), C.c_int, C.POINTER(C.c_void_p)]),
    "ttg_mps_from_device": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.POINTER(C.c_void_p), C.POINTER(C.c_double),
                                      C.POINTER(C.c_void_p)]),
    "ttg_mps_free": (None, [C.c_void_p]),
    "ttg_mps_info": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                               C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_double),
                               C.POINTER(C.c_int)]),
    "ttg_mps_download": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "ttg_mps_download_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ttg_mps_site_ptr": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "ttg_mpo_upload": (C.c_int, [C.c_void_p, C.POINTER(ttg_mpo_view), C.POINTER(C.c_void_p)]),
    "ttg_mpo_free": (None, [C.c_void_p]),
    "ttg_apply_raw": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ttg_hadamard": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "ttg_simplify": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(ttg_strategy), C.c_void_p,
                               C.POINTER(C.c_void_p), C.POINTER(ttg_report)]),
    "ttg_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(ttg_strategy), C.POINTER(C.c_void_p),
                            C.POINTER(ttg_report)]),
    "ttg_canonicalize": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(ttg_strategy),
                                   C.POINTER(C.c_void_p), C.POINTER(ttg_report)]),
    "ttg_recenter": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(ttg_strategy),
                               C.POINTER(C.c_void_p), C.POINTER(C.c_double)]),
    "ttg_schmidt_split": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_void_p, C.c_int,
                                    C.POINTER(ttg_strategy), C.c_void_p, C.c_void_p, C.POINTER(C.c_int64),
                                    C.POINTER(C.c_double)]),
    "ttg_mps_join": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "ttg_simplify_sum": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                    C.POINTER(C.c_void_p), C.POINTER(ttg_strategy), C.c_void_p,
                                    C.POINTER(C.c_void_p), C.POINTER(ttg_report)]),
    "ttg_mps_load": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "ttg_mps_save": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_char_p]),
    "ttg_mpo_load": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "ttg_mpo_save": (C.c_int, [C.c_void_p, C.c_void_p, C.c_char_p]),
    "ttg_expectation_mpo": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double)]),
    "ttg_scprod": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "ttg_apply_effective_two_site": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ttg_apply_effective_two_site_dev": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ttg_op_env_update": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p]),
    "ttg_debug_gemm": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                 C.c_void_p, C.c_void_p]),
    "ttg_debug_gemm_dev": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_double)]),
    "ttg_debug_svd": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_int64, C.c_void_p,
                                C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "ttg_debug_svd_ex": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_int64,
                                   C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                   C.POINTER(C.c_int), C.POINTER(C.c_double), C.c_double]),
    "ttg_debug_qr": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ttg_debug_qr_blocked": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ttg_debug_qr_pre": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                    C.POINTER(C.c_double)]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"ttgpu native library missing: {path} (run __graft_entry__.build() / make)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = load()
