"""``ModelConfig`` — the same fields, defaults, derived sizes and validation rules as the
reference (``pkg/src/longrec/config.py:19-96``), plus the device-path limits of this build.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass, fields

from .errors import ConfigError

QUERY_STRATEGIES = ("recent", "uniform", "learnable", "recent_uniform")
MERGE_MODES = ("concat", "inner")


@dataclass
class ModelConfig:
    L: int = 256                 # visible raw sequence length
    d: int = 8                   # per-item token width
    K: int = 4                   # merge group size
    m: int = 3                   # global tokens: UID, CLS..., target
    k: int = 16                  # sampled sequence queries
    N: int = 2                   # self-attention layers after the cross layer
    heads: int = 1
    merge_mode: str = "concat"   # "concat" | "inner"
    inner_layers: int = 1
    query_strategy: str = "recent"
    head_hidden: int = 32
    d_item: int = 8
    d_act: int = 4
    d_time: int = 8
    n_time_buckets: int = 32
    vocab: int = 200
    n_actions: int = 4
    n_users: int = 4000
    n_profiles: int = 16
    lr: float = 3e-3
    batch_size: int = 32

    @property
    def D(self) -> int:
        return self.K * self.d

    @property
    def feat_width(self) -> int:
        return self.d_item + self.d_act + self.d_time

    @property
    def L_padded(self) -> int:
        return -(-self.L // self.K) * self.K

    @property
    def merged_len(self) -> int:
        return self.L_padded // self.K

    def validate(self) -> "ModelConfig":
        """Reference rules (pkg/src/longrec/config.py:68-89)."""
        if self.L < 1 or self.d < 1 or self.K < 1:
            raise ConfigError("L, d, K must all be >= 1")
        if self.m < 3:
            raise ConfigError("m must be >= 3 (UID, at least one CLS, target)")
        if self.N < 1:
            raise ConfigError("N must be >= 1")
        if self.k < 1:
            raise ConfigError("k must be >= 1")
        if self.query_strategy not in QUERY_STRATEGIES:
            raise ConfigError(f"unknown query_strategy {self.query_strategy!r}")
        if self.merge_mode not in MERGE_MODES:
            raise ConfigError(f"unknown merge_mode {self.merge_mode!r}")
        if self.query_strategy != "learnable" and self.k > self.merged_len:
            raise ConfigError(
                f"k={self.k} exceeds merged length {self.merged_len} for token-sampling strategies")
        if self.D % self.heads:
            raise ConfigError(f"width D={self.D} not divisible by heads={self.heads}")
        if self.inner_layers < 1:
            raise ConfigError("inner_layers must be >= 1")
        return self

    def to_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, payload: dict) -> "ModelConfig":
        if not isinstance(payload, dict):
            raise ConfigError("ModelConfig payload must be a JSON object")
        known = {f.name for f in fields(cls)}
        for key in payload:
            if key not in known:
                raise ConfigError(f"unknown config field {key!r} for ModelConfig")
        return cls(**payload).validate()
