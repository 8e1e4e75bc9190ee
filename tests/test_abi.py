"""The C-ABI library loads on CPU and exports every symbol include/ttgpu.h declares."""
import os
import re

from paper_2601_16734_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "ttgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(ttg_[a-z0-9_]+)\s*\(", src))


def test_header_symbols_exported():
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(_lib.lib, n), n
    assert names == set(_lib.SIGNATURES), names ^ set(_lib.SIGNATURES)


def test_no_device_is_an_error_not_a_fallback():
    import ctypes as C
    import torch
    if torch.cuda.is_available():
        return
    h = C.c_void_p()
    assert _lib.lib.ttg_create(0, C.byref(h)) == _lib.TTG_CUDA
    assert _lib.lib.ttg_version().startswith(b"ttgpu")
