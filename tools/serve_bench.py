"""Serving throughput on one GPU (not the headline bench): per-user cache build and batched
candidate scoring against the full forward of the same (user, candidate) pairs.

    python tools/serve_bench.py [--config c2_inner] [--users 64] [--cands 512]

Prints one JSON line: cache build users/s, cached scoring candidates/s, full-forward
candidates/s (each a median of CUDA-event-timed repetitions, inputs resident in HBM).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import CONFIGS  # noqa: E402
from paper_2505_04421_b200 import ModelConfig, serving as S  # noqa: E402
from paper_2505_04421_b200.inputs import Batch, synthetic_batch  # noqa: E402
from paper_2505_04421_b200.model import LongerModel  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2_inner")
    ap.add_argument("--users", type=int, default=64)
    ap.add_argument("--cands", type=int, default=512)
    args = ap.parse_args()
    cfg = ModelConfig(**CONFIGS[args.config]).validate()
    U, C = args.users, args.cands
    model = LongerModel(cfg, seed=0)
    users = synthetic_batch(cfg, U, seed=3).to("cuda")
    cand = torch.randint(0, cfg.vocab, (U, C), dtype=torch.int32, device="cuda")
    times = [0] * U
    cache = S.build_caches_batch(model, users, times)
    ms_build = timed(lambda: S.build_caches_batch(model, users, times), reps=5)
    ms_score = timed(lambda: S.score_candidates(model, cache, cand, check=False))
    # full forward of the same pairs, in batches of 256 samples
    rep = lambda a: a.repeat_interleave(C, dim=0)
    full = Batch(rep(users.items), rep(users.actions), rep(users.dt), rep(users.n_events), rep(users.uid),
                 rep(users.profile), cand.reshape(-1).contiguous(), torch.zeros(U * C, device="cuda"))
    nb = min(256, U * C)
    sub = Batch(*[getattr(full, f)[:nb].contiguous() for f in Batch.FIELDS])
    ms_full = timed(lambda: model.forward(sub), reps=5)
    p_c = S.score_candidates(model, cache, cand).reshape(-1)[:nb]
    p_f = model.forward(sub)
    print(json.dumps({
        "config": args.config, "users": U, "candidates_per_user": C,
        "cache_build_ms": round(ms_build, 3), "cache_build_users_per_s": round(U / ms_build * 1e3, 1),
        "cache_bytes_per_user": S.cache_size_bytes(model, 1),
        "score_ms": round(ms_score, 3), "cached_candidates_per_s": round(U * C / ms_score * 1e3, 1),
        "full_forward_candidates_per_s": round(nb / ms_full * 1e3, 1),
        "max_abs_cached_minus_full": float((p_c - p_f).abs().max()),
    }))


if __name__ == "__main__":
    main()
