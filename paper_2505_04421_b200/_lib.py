"""ctypes binding of the sm_100a C-ABI library (``include/longer.h``).

The product path has no CPU fallback: if the library is missing, the device is not a CUDA
device, or a call fails, this module raises.  Status codes map 1:1 onto the reference
exception classes (``pkg/src/longrec/errors.py:8-29``).
"""
from __future__ import annotations

import ctypes
from pathlib import Path

from .errors import (ConfigError, DimensionError, EmbeddingLookupError, NumericalError,
                     StaleCacheError)

_PKG = Path(__file__).resolve().parent
_SO = _PKG / "_longer_sm100.so"
_lib = None

LONGER_OK, LONGER_ECONFIG, LONGER_EDIM, LONGER_ELOOKUP, LONGER_ENUMERIC, LONGER_ESTALE, LONGER_ECUDA = range(7)
_EXC = {LONGER_ECONFIG: ConfigError, LONGER_EDIM: DimensionError, LONGER_ELOOKUP: EmbeddingLookupError,
        LONGER_ENUMERIC: NumericalError, LONGER_ESTALE: StaleCacheError, LONGER_ECUDA: RuntimeError}

SYMBOLS = ("longer_param_count", "longer_workspace_bytes", "longer_forward", "longer_forward_backward",
           "longer_adam_step", "longer_read_status", "longer_last_error", "longer_set_probe",
           "longer_cache_bytes", "longer_cache_build", "longer_score_workspace_bytes", "longer_cache_score",
           "longer_backward", "longer_forward_trace", "longer_grad_early_begin", "longer_set_grad_event")

PROBES = {"fe_fwd": 0, "fe_inner_bwd": 1, "fe_mlp_bwd": 2, "xattn_fwd": 3, "xattn_bwd": 4,
          "fwd_rows": 5, "bwd_rows": 6}   # the last two bracket sections, not single kernels


class LongerDims(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "L", "d", "K", "m", "k", "N", "heads", "merge_inner", "inner_layers", "query_strategy",
        "head_hidden", "d_item", "d_act", "d_time", "n_time_buckets", "vocab", "n_actions",
        "n_users", "n_profiles", "batch")]


class LongerBatch(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in (
        "items", "actions", "dt", "n_events", "uid", "profile", "cand_item", "label")]


class LongerTrace(ctypes.Structure):
    _fields_ = [("h", ctypes.c_void_p), ("merged", ctypes.c_void_p), ("query_groups", ctypes.c_void_p),
                ("layers", ctypes.c_void_p * 17), ("head_input", ctypes.c_void_p),
                ("n_layers", ctypes.c_int32), ("Lp", ctypes.c_int32), ("G", ctypes.c_int32),
                ("q", ctypes.c_int32), ("head_width", ctypes.c_int32)]


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
    lib = ctypes.CDLL(str(_SO), mode=ctypes.RTLD_GLOBAL)
    _declare(lib)
    _lib = lib
    return lib


def _declare(lib):
    vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float
    pd, pb = ctypes.POINTER(LongerDims), ctypes.POINTER(LongerBatch)
    sig = {
        "longer_param_count": [pd, ctypes.POINTER(i64)],
        "longer_workspace_bytes": [pd, ctypes.POINTER(ctypes.c_size_t)],
        "longer_forward": [pd, vp, pb, vp, ctypes.c_size_t, vp, vp],
        "longer_forward_backward": [pd, vp, pb, vp, ctypes.c_size_t, vp, vp, vp, vp],
        "longer_backward": [pd, vp, pb, vp, ctypes.c_size_t, vp, vp, vp, vp],
        "longer_forward_trace": [pd, vp, pb, vp, ctypes.c_size_t, vp, ctypes.POINTER(LongerTrace), vp],
        "longer_adam_step": [vp, vp, vp, vp, i64, f32, i32, vp],
        "longer_read_status": [vp, ctypes.POINTER(i32), vp],
        "longer_set_probe": [i32, vp, vp],
        "longer_grad_early_begin": [pd, ctypes.POINTER(i64)],
        "longer_set_grad_event": [vp],
        "longer_cache_bytes": [pd, ctypes.POINTER(ctypes.c_size_t)],
        "longer_cache_build": [pd, vp, pb, vp, ctypes.c_size_t, vp, ctypes.c_size_t, vp],
        "longer_score_workspace_bytes": [pd, i32, ctypes.POINTER(ctypes.c_size_t)],
        "longer_cache_score": [pd, vp, vp, ctypes.c_size_t, vp, i32, vp, ctypes.c_size_t, vp, vp],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.restype = ctypes.c_int
        fn.argtypes = args
    lib.longer_last_error.restype = ctypes.c_char_p
    lib.longer_last_error.argtypes = []
    if hasattr(lib, "longer_test_gemm"):
        lib.longer_test_gemm.restype = ctypes.c_int
        lib.longer_test_gemm.argtypes = [vp, i32, i32, vp, i32, i32, vp, i32, i32, i32, i32, vp]
    if hasattr(lib, "longer_test_layernorm"):
        lib.longer_test_layernorm.restype = ctypes.c_int
        lib.longer_test_layernorm.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp]


def check(rc: int) -> None:
    if rc == LONGER_OK:
        return
    msg = _lib.longer_last_error().decode() if _lib is not None else ""
    raise _EXC.get(rc, RuntimeError)(msg or f"longer error {rc}")


def dims_of(cfg, batch: int) -> LongerDims:
    from .config import QUERY_STRATEGIES
    return LongerDims(L=cfg.L, d=cfg.d, K=cfg.K, m=cfg.m, k=cfg.k, N=cfg.N, heads=cfg.heads,
                      merge_inner=1 if cfg.merge_mode == "inner" else 0,
                      inner_layers=cfg.inner_layers, query_strategy=QUERY_STRATEGIES.index(cfg.query_strategy),
                      head_hidden=cfg.head_hidden, d_item=cfg.d_item, d_act=cfg.d_act, d_time=cfg.d_time,
                      n_time_buckets=cfg.n_time_buckets, vocab=cfg.vocab, n_actions=cfg.n_actions,
                      n_users=cfg.n_users, n_profiles=cfg.n_profiles, batch=batch)
