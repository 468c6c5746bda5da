"""Generate golden vectors by running the REFERENCE implementation (longrec) itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

For each case it builds ``LongRecModel(cfg, seed)``, a list of ``Sample``s, and records
  * the model parameters by name (float64),
  * the tensorised batch (the C-ABI layout, see paper_2505_04421_b200/inputs.py),
  * per-sample probabilities from ``model.forward`` (pkg/src/longrec/model.py:365-372),
  * the batch-mean BCE and every parameter gradient of the training-step body
    (zero_grads → per-sample ``T.bce(forward_tensor)`` → ``T.mean_scalars`` → backward,
    pkg/src/longrec/model.py:555-567),
into ``tests/golden/<case>.npz``.  These files are committed; the GPU box never needs
/root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from longrec import tensors as T  # noqa: E402
from longrec.config import ModelConfig as RefConfig  # noqa: E402
from longrec.inputs import Candidate, Event, Sample, UserFeatures  # noqa: E402
from longrec.model import LongRecModel  # noqa: E402

from paper_2505_04421_b200 import inputs as I  # noqa: E402
from paper_2505_04421_b200.config import ModelConfig  # noqa: E402

TINY = dict(L=8, d=2, K=2, m=3, k=3, N=2, heads=1, d_item=3, d_act=2, d_time=2, n_time_buckets=8,
            vocab=12, n_actions=3, n_users=6, n_profiles=4, head_hidden=5)

CASES = {
    "tiny_concat": (dict(TINY), [8, 6, 3, 0, 12, 1], 5),
    "tiny_inner2": (dict(TINY, merge_mode="inner", inner_layers=2), [8, 6, 3, 0, 12, 1], 6),
    "tiny_heads2_m4": (dict(TINY, d=4, heads=2, m=4, merge_mode="inner"), [8, 5, 2, 7], 7),
    "tiny_oddL": (dict(TINY, L=7, merge_mode="inner"), [7, 4, 1, 9], 8),
    "small_c1": (dict(L=64, d=16, K=4, k=16, N=1, m=3, n_users=64), [64, 64, 40, 10, 64], 9),
    "small_c2_inner": (dict(L=64, d=32, K=4, k=8, N=2, m=3, merge_mode="inner", n_users=64), [64, 50, 64, 3], 10),
    # device-eligible (d % 8 == 0) edge cases: odd L, heads=2, m=4, two inner layers, pad queries
    "gpu_d8_h2": (dict(L=30, d=8, K=4, m=4, k=5, N=2, heads=2, merge_mode="inner", inner_layers=2,
                       head_hidden=16, n_users=50, vocab=60), [30, 17, 5, 0, 40, 12], 11),
    "gpu_concat_d8": (dict(L=48, d=8, K=2, k=6, N=3, n_users=40), [48, 20, 3, 48], 12),
    # the other query strategies (pkg/src/longrec/model.py:58-123): non-contiguous query groups,
    # pad queries when fewer than k non-pad groups exist, a learned query bank
    "qs_uniform": (dict(TINY, L=30, K=2, k=5, query_strategy="uniform"), [30, 17, 9, 4, 0], 13),
    "qs_recent_uniform": (dict(TINY, L=30, K=2, k=5, query_strategy="recent_uniform"), [30, 17, 9, 4, 0], 14),
    "qs_learnable": (dict(TINY, L=30, K=2, k=5, query_strategy="learnable", merge_mode="inner"), [30, 11, 2, 0], 15),
    "gpu_d8_uniform": (dict(L=64, d=8, K=4, m=4, k=6, N=2, heads=2, merge_mode="inner", query_strategy="uniform",
                            head_hidden=16, n_users=50, vocab=60), [64, 41, 13, 5, 0], 16),
    "gpu_d8_recent_uniform": (dict(L=64, d=8, K=2, m=3, k=7, N=2, query_strategy="recent_uniform",
                                   n_users=50, vocab=60), [64, 30, 11, 64], 17),
    "gpu_d8_learnable": (dict(L=48, d=8, K=4, m=3, k=5, N=2, query_strategy="learnable", merge_mode="inner",
                              n_users=50, vocab=60), [48, 20, 3, 0], 18),
}


def make_samples(cfg, n_events_list, seed):
    rng = np.random.default_rng(seed)
    out = []
    for i, n in enumerate(n_events_list):
        t = 1_700_000_000
        ev = []
        for j in range(n):
            gap = int(rng.integers(30, 900))
            if i == 1 and j == 1:
                gap = 2 ** 40          # the oldest event lies > 2^40 s before the candidate → bucket clamp
            t += gap
            ev.append(Event(int(rng.integers(cfg["vocab"] if "vocab" in cfg else 200)),
                            int(rng.integers(cfg.get("n_actions", 4))), t))
        if i == 2 and n > 1:          # equal timestamps (delta 0 → bucket 0)
            ev[-1] = Event(ev[-1].item_id, ev[-1].action_type, ev[-1].timestamp)
        cand_ts = t + (0 if i == 2 else 60)
        uid = int(rng.integers(cfg.get("n_users", 4000)))
        prof = int(rng.integers(cfg.get("n_profiles", 16)))
        out.append(Sample(tuple(ev), UserFeatures(uid, prof),
                          Candidate(int(rng.integers(cfg.get("vocab", 200))), cand_ts), i % 2))
    return out


def run_case(name, cfg_kw, n_list, seed):
    rcfg = RefConfig(**cfg_kw).validate()
    cfg = ModelConfig(**cfg_kw).validate()
    model = LongRecModel(rcfg, seed=seed)
    samples = make_samples(cfg_kw, n_list, seed + 100)
    p = np.array([model.forward(s)[0] for s in samples])
    for _, t in model.params():
        t.zero_grad()
    losses = [T.bce(model.forward_tensor(s), s.label) for s in samples]
    loss = T.mean_scalars(losses)
    loss.backward()
    # the tensorised batch uses our mirror records (same field values)
    mine = [I.Sample(tuple(I.Event(e.item_id, e.action_type, e.timestamp) for e in s.events),
                     I.UserFeatures(s.user_features.uid, s.user_features.profile_bucket),
                     I.Candidate(s.candidate.item_id, s.candidate.timestamp), s.label) for s in samples]
    b = I.tensorize(mine, cfg)
    arrays = {"cfg": np.array(json.dumps(cfg.to_dict())), "p": p, "loss": np.array(float(loss.data)),
              "seed": np.array(seed)}
    for f in I.Batch.FIELDS:
        arrays["batch/" + f] = getattr(b, f)
    for n, t in model.params():
        arrays["P/" + n] = t.data
        arrays["G/" + n] = np.zeros_like(t.data) if t.grad is None else t.grad
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}: B={len(samples)} loss={float(loss.data):.6f} -> {os.path.relpath(path, ROOT)}")


if __name__ == "__main__":
    for name, (kw, n_list, seed) in CASES.items():
        run_case(name, kw, n_list, seed)
