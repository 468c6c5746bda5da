"""``LRCKPT01`` weight interchange (pkg/src/longrec/model.py:381-427), NumPy-only.

Layout: 8-byte magic ``LRCKPT01``; uint64 LE header length; UTF-8 JSON header
{format_version: 1, config, param_version, arrays: [{name, shape}]} (sorted keys); then each
array's float64 little-endian bytes in header order.  Adam moments are not part of the format
(the reference does not save them either).
"""
from __future__ import annotations

import json
import struct

import numpy as np

from .config import ModelConfig
from .errors import ConfigError
from .params import param_shapes

MAGIC = b"LRCKPT01"


def write_checkpoint(path: str, cfg: ModelConfig, named, param_version: int = 0) -> None:
    named = [(n, np.asarray(a, dtype=np.float64)) for n, a in named]
    header = {"format_version": 1, "config": cfg.to_dict(), "param_version": int(param_version),
              "arrays": [{"name": n, "shape": list(a.shape)} for n, a in named]}
    blob = json.dumps(header, sort_keys=True).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<Q", len(blob)))
        fh.write(blob)
        for _, a in named:
            fh.write(a.astype("<f8").tobytes())


def read_checkpoint(path: str):
    """→ (cfg, {name: float64 array}, param_version); validates names and shapes."""
    with open(path, "rb") as fh:
        magic = fh.read(8)
        if magic != MAGIC:
            raise ConfigError(f"not a checkpoint file: bad magic {magic!r}")
        (hlen,) = struct.unpack("<Q", fh.read(8))
        header = json.loads(fh.read(hlen).decode("utf-8"))
        if header.get("format_version") != 1:
            raise ConfigError("unsupported checkpoint format version")
        cfg = ModelConfig.from_dict(header["config"])
        shapes = param_shapes(cfg)
        out = {}
        for entry in header["arrays"]:
            name, shape = entry["name"], tuple(entry["shape"])
            if name not in shapes:
                raise ConfigError(f"checkpoint array {name!r} not in model")
            if tuple(shapes[name]) != shape:
                raise ConfigError(f"checkpoint array {name!r} shape mismatch")
            count = int(np.prod(shape)) if shape else 1
            out[name] = np.frombuffer(fh.read(count * 8), dtype="<f8").reshape(shape).copy()
    return cfg, out, int(header["param_version"])
