"""CPU checks of bench.py's serving (c4) accounting: the MAC model restates the reference's
muladds_cache_build / muladds_incremental (pkg/src/longrec/analysis.py:174-198)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_serve_macs_match_reference_model():
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present (GPU box)")
    sys.path.insert(0, ref)
    from longrec import analysis, config as rc
    from bench import CONFIGS, serve_macs
    from paper_2505_04421_b200 import ModelConfig
    for name in ("c2_inner", "c2_concat", "c1"):
        kw = CONFIGS[name]
        cfg = ModelConfig(**kw).validate()
        rcfg = rc.ModelConfig(**kw).validate()
        build, inc = serve_macs(cfg)
        assert build == analysis.muladds_cache_build(rcfg, cfg.L)
        assert inc == analysis.muladds_incremental(rcfg)
