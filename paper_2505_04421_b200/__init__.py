"""B200-native (sm_100a) LONGER encoder — drop-in for the reference ``longrec`` hot path.

Public surface mirrors ``longrec`` (pkg/src/longrec/__init__.py:12-31) for the encoder path:
``ModelConfig``, ``Sample``/``Event``/``UserFeatures``/``Candidate``, ``LongerModel`` (alias
``LongRecModel``), ``Adam``, and the reference exception classes.
"""
from .config import ModelConfig
from .errors import (ConfigError, DimensionError, EmbeddingLookupError, NumericalError,
                     StaleCacheError, UndefinedMetricError)
from .inputs import Batch, Candidate, Event, Sample, UserFeatures, synthetic_batch, synthetic_samples, tensorize
from .params import count_params, init_params, param_shapes

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent pieces load lazily so that config/oracle tooling imports without CUDA
    if name in ("LongerModel", "LongRecModel"):
        from .model import LongerModel
        return LongerModel
    if name == "Adam":
        from .model import Adam
        return Adam
    raise AttributeError(name)


__all__ = ["ModelConfig", "ConfigError", "DimensionError", "EmbeddingLookupError", "NumericalError",
           "StaleCacheError", "UndefinedMetricError", "Batch", "Candidate", "Event", "Sample", "UserFeatures",
           "synthetic_batch", "synthetic_samples", "tensorize", "count_params", "init_params", "param_shapes",
           "LongerModel", "LongRecModel", "Adam"]
