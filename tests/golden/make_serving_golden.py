"""Generate serving golden vectors with the REFERENCE two-stage path (longrec.serving).

Run in the build container (where /root/reference exists):

    python tests/golden/make_serving_golden.py

For each case: ``LongRecModel(cfg, seed)``, a few users (events, features, scoring time) and C
candidates per user; records the parameters, every user's history tensorised with the scoring
time as the time reference (the C-ABI batch layout), the candidate ids and the probabilities of
``score_with_cache(model, build_cache(...), candidate)`` (pkg/src/longrec/serving.py:84-167),
plus the full-forward probabilities of the same (user, candidate) samples for comparison.
Output: ``tests/golden/serving_<case>.npz`` (committed; the GPU box never reads /root/reference).
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

from longrec.config import ModelConfig as RefConfig  # noqa: E402
from longrec.inputs import Candidate, Event, Sample, UserFeatures  # noqa: E402
from longrec.model import LongRecModel  # noqa: E402
from longrec.serving import build_cache, score_with_cache  # noqa: E402

from paper_2505_04421_b200 import inputs as I  # noqa: E402
from paper_2505_04421_b200.config import ModelConfig  # noqa: E402

CASES = {
    # inner merge, two heads, m=4, a user with no events and one shorter than k groups
    "serving_d8_inner_h2": (dict(L=30, d=8, K=4, m=4, k=5, N=2, heads=2, merge_mode="inner",
                                 head_hidden=16, n_users=50, vocab=60), [30, 11, 0, 2], 5, 21),
    # concat merge, three self layers
    "serving_d8_concat": (dict(L=48, d=8, K=2, k=6, N=3, n_users=40, vocab=80), [48, 20, 7], 6, 22),
    # c1-like widths at a short L
    "serving_d16_c1": (dict(L=64, d=16, K=4, k=16, N=1, m=3, n_users=64), [64, 40, 9], 4, 23),
}


def run_case(name, cfg_kw, n_list, C, seed):
    rcfg = RefConfig(**cfg_kw).validate()
    cfg = ModelConfig(**cfg_kw).validate()
    model = LongRecModel(rcfg, seed=seed)
    rng = np.random.default_rng(seed + 100)
    users, cands, p_cached, p_full = [], [], [], []
    for n in n_list:
        t = 1_700_000_000
        ev = []
        for _ in range(n):
            t += int(rng.integers(30, 900))
            ev.append(Event(int(rng.integers(rcfg.vocab)), int(rng.integers(rcfg.n_actions)), t))
        feats = UserFeatures(int(rng.integers(rcfg.n_users)), int(rng.integers(rcfg.n_profiles)))
        scoring_time = t + 120
        cache = build_cache(model, tuple(ev), feats, scoring_time)
        row, pc, pf = [], [], []
        for _ in range(C):
            cand = Candidate(int(rng.integers(rcfg.vocab)), scoring_time)
            row.append(cand.item_id)
            pc.append(score_with_cache(model, cache, cand))
            pf.append(float(model.forward(Sample(tuple(ev), feats, cand, 0))[0]))
        users.append(I.Sample(tuple(I.Event(e.item_id, e.action_type, e.timestamp) for e in ev),
                              I.UserFeatures(feats.uid, feats.profile_bucket), I.Candidate(0, scoring_time), 0))
        cands.append(row)
        p_cached.append(pc)
        p_full.append(pf)
    b = I.tensorize(users, cfg)
    arrays = {"cfg": np.array(json.dumps(cfg.to_dict())), "cand": np.array(cands, np.int32),
              "p_cached": np.array(p_cached), "p_full": np.array(p_full), "seed": np.array(seed),
              "scoring_time": np.array([u.candidate.timestamp for u in users], np.int64)}
    for f in I.Batch.FIELDS:
        arrays["users/" + f] = getattr(b, f)
    for n, t in model.params():
        arrays["P/" + n] = t.data
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    dev = float(np.max(np.abs(np.array(p_cached) - np.array(p_full))))
    print(f"{name}: U={len(users)} C={C} max|cached-full|={dev:.2e} -> {os.path.relpath(path, ROOT)}")


if __name__ == "__main__":
    for name, (kw, n_list, C, seed) in CASES.items():
        run_case(name, kw, n_list, C, seed)
