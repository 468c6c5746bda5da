"""LRCKPT01 interchange: our writer/reader round-trip, and compatibility with the reference
reader/writer when /root/reference is present (build container only; skipped elsewhere)."""
import os
import sys

import numpy as np
import pytest

from paper_2505_04421_b200 import ModelConfig, init_params
from paper_2505_04421_b200.checkpoint import read_checkpoint, write_checkpoint
from paper_2505_04421_b200.errors import ConfigError

REF = "/root/reference/pkg/src"


def test_roundtrip(tmp_path):
    cfg = ModelConfig(L=16, d=8, K=2, k=4, merge_mode="inner").validate()
    P = init_params(cfg, 3)
    write_checkpoint(tmp_path / "a.ckpt", cfg, P.items(), 7)
    cfg2, Q, v = read_checkpoint(tmp_path / "a.ckpt")
    assert cfg2 == cfg and v == 7 and list(Q) == list(P)
    for n in P:
        np.testing.assert_array_equal(P[n], Q[n])


def test_bad_magic(tmp_path):
    (tmp_path / "x").write_bytes(b"NOTACKPT" + b"\0" * 16)
    with pytest.raises(ConfigError):
        read_checkpoint(tmp_path / "x")


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
def test_reference_reads_ours_and_we_read_reference(tmp_path):
    sys.path.insert(0, REF)
    from longrec.config import ModelConfig as RC
    from longrec.model import LongRecModel
    kw = dict(L=16, d=8, K=2, k=4, merge_mode="inner")
    cfg = ModelConfig(**kw).validate()
    P = init_params(cfg, 5)
    write_checkpoint(tmp_path / "ours.ckpt", cfg, P.items(), 2)
    ref = LongRecModel.load(str(tmp_path / "ours.ckpt"))
    assert ref.param_version == 2
    for n, t in ref.params():
        np.testing.assert_array_equal(t.data, P[n])
    ref2 = LongRecModel(RC(**kw), seed=9)
    ref2.save(str(tmp_path / "ref.ckpt"))
    _, Q, _ = read_checkpoint(tmp_path / "ref.ckpt")
    for n, t in ref2.params():
        np.testing.assert_array_equal(t.data, Q[n])
