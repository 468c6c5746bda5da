"""JSONL dataset I/O mirrors pkg/src/longrec/inputs.py:279-301 (same record layout, same errors),
and the host batches it yields carry exactly the samples' fields (CPU)."""
import os
import sys

import numpy as np
import pytest

from paper_2505_04421_b200 import ConfigError, ModelConfig, synthetic_samples
from paper_2505_04421_b200.inputs import (Candidate, Dataset, Event, Sample, UserFeatures, load_dataset,
                                          save_dataset, tensorize)

REF = "/root/reference/pkg/src"


def test_round_trip(tmp_path):
    cfg = ModelConfig(L=64, d=16, K=4, k=8, N=1, m=3).validate()
    ds = Dataset(synthetic_samples(cfg, 7, seed=3))
    for name in ("a.jsonl", "b.jsonl.gz"):
        path = str(tmp_path / name)
        save_dataset(ds, path)
        back = load_dataset(path, L_max=cfg.L)
        assert back.samples == ds.samples
        batches = list(back.batches(cfg, 3, pin=False))
        assert [b.size for b in batches] == [3, 3, 1]
        ref = tensorize(ds.samples, cfg)
        np.testing.assert_array_equal(np.concatenate([b.items for b in batches]), ref.items)


def test_validation_errors(tmp_path):
    bad = Sample((Event(1, 0, 10), Event(2, 0, 5)), UserFeatures(0, 0), Candidate(1, 20), 0)
    with pytest.raises(ConfigError):
        bad.validate()
    path = tmp_path / "m.jsonl"
    path.write_text('{"events": [], "label": 0}\n')
    with pytest.raises(ConfigError):
        load_dataset(str(path))


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference checkout not present")
def test_reads_and_writes_the_reference_format(tmp_path):
    sys.path.insert(0, REF)
    from longrec import inputs as RI
    cfg = ModelConfig(L=32, d=8, K=2, k=4, N=1, m=3).validate()
    ours = synthetic_samples(cfg, 5, seed=8)
    p1 = str(tmp_path / "ours.jsonl")
    save_dataset(Dataset(ours), p1)
    theirs = RI.load_dataset(p1, L_max=cfg.L)                # reference reads our file
    assert [s.to_json_dict() for s in theirs.samples] == [s.to_json_dict() for s in ours]
    p2 = str(tmp_path / "theirs.jsonl.gz")
    RI.save_dataset(theirs, p2)                              # we read the reference's file
    assert load_dataset(p2).samples == ours


def test_vectorised_tensorize_matches_per_sample_layout():
    """tensorize places every sample's last L events right-aligned, with deltas from its own
    candidate timestamp (encode_events, pkg/src/longrec/inputs.py:457-482)."""
    cfg = ModelConfig(L=16, d=16, K=4, k=2, N=1, m=3).validate()
    smp = synthetic_samples(cfg, 5, seed=9, n_events=30)[:2] + synthetic_samples(cfg, 3, seed=4, n_events=7)
    b = tensorize(smp, cfg)
    for i, s in enumerate(smp):
        ev = s.events[-cfg.L:]
        n = len(ev)
        assert b.n_events[i] == n
        np.testing.assert_array_equal(b.items[i, cfg.L - n:], [e.item_id for e in ev])
        np.testing.assert_array_equal(b.actions[i, cfg.L - n:], [e.action_type for e in ev])
        np.testing.assert_array_equal(b.dt[i, cfg.L - n:], [s.candidate.timestamp - e.timestamp for e in ev])
        assert not b.items[i, :cfg.L - n].any() and not b.dt[i, :cfg.L - n].any()


def test_dataset_batches_slice_the_tensorised_dataset():
    cfg = ModelConfig(L=16, d=16, K=4, k=2, N=1, m=3).validate()
    ds = Dataset(synthetic_samples(cfg, 11, seed=2, n_events=9))
    full = tensorize(ds.samples, cfg)
    got = list(ds.batches(cfg, 4, pin=False))
    assert [g.size for g in got] == [4, 4, 3]
    np.testing.assert_array_equal(np.concatenate([g.items for g in got]), full.items)
    sh = list(ds.batches(cfg, 4, pin=False, shuffle=True, seed=1))
    assert sorted(np.concatenate([g.uid for g in sh]).tolist()) == sorted(full.uid.tolist())
