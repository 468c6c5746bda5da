"""ctypes binding of the sm_100a C-ABI library (``include/longer.h``).

The product path has no CPU fallback: if the library is missing or the device is not
sm_100, :func:`load` raises.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
_SO = _PKG / "_longer_sm100.so"
_lib = None


def so_path() -> Path:
    return _SO


def load(build_if_missing: bool = True):
    global _lib
    if _lib is not None:
        return _lib
    if not _SO.exists():
        if not build_if_missing:
            raise RuntimeError(f"sm_100a library {_SO} is missing; run __graft_entry__.build()")
        from . import build as _build
        _build.build()
    _lib = ctypes.CDLL(str(_SO), mode=ctypes.RTLD_GLOBAL)
    _declare(_lib)
    return _lib


def _declare(lib):
    vp, i32 = ctypes.c_void_p, ctypes.c_int
    if hasattr(lib, "longer_test_gemm"):
        lib.longer_test_gemm.restype = i32
        lib.longer_test_gemm.argtypes = [vp, i32, i32, vp, i32, i32, vp, i32, i32, i32, i32, vp]
