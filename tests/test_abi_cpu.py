"""CPU-side checks of the boundary: the library loads, exports every symbol include/longer.h
declares, and its parameter layout / validation agree with the host mirror (no GPU work)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2505_04421_b200 import ModelConfig, _lib
from paper_2505_04421_b200.errors import ConfigError
from paper_2505_04421_b200.params import count_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "longer.h")).read()
    return sorted(set(re.findall(r"\b(longer_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert set(syms) == set(_lib.SYMBOLS)
    for s in syms:
        assert hasattr(lib, s), s


@pytest.mark.parametrize("kw", [dict(), dict(L=2000, d=32, K=4, k=32, N=2, merge_mode="inner"),
                                dict(L=30, d=8, K=4, m=4, k=5, N=2, heads=2, merge_mode="inner", inner_layers=2)])
def test_param_count_matches_host_layout(kw):
    cfg = ModelConfig(**kw).validate()
    lib = _lib.load()
    n = ctypes.c_int64()
    _lib.check(lib.longer_param_count(ctypes.byref(_lib.dims_of(cfg, 1)), ctypes.byref(n)))
    assert n.value == count_params(cfg)
    ws = ctypes.c_size_t()
    _lib.check(lib.longer_workspace_bytes(ctypes.byref(_lib.dims_of(cfg, 8)), ctypes.byref(ws)))
    assert ws.value > 0


def test_library_rejects_bad_config_with_reference_error():
    lib = _lib.load()
    cfg = ModelConfig(d=4)   # d % 8 != 0 is outside the device path
    n = ctypes.c_int64()
    with pytest.raises(ConfigError):
        _lib.check(lib.longer_param_count(ctypes.byref(_lib.dims_of(cfg, 1)), ctypes.byref(n)))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2505_04421_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), f
