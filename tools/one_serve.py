"""One cached-scoring call (c4: 64 users x 512 candidates) inside cudaProfilerStart/Stop after
warm-up, for `ncu --profile-from-start off` launch lists."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2505_04421_b200 import ModelConfig, serving as S, synthetic_batch  # noqa: E402
from paper_2505_04421_b200.model import LongerModel  # noqa: E402

cfg = ModelConfig(**CONFIGS["c2_inner"]).validate()
U, C = 64, 512
model = LongerModel(cfg, seed=0)
users = synthetic_batch(cfg, U, seed=3).to("cuda")
cache = S.build_caches_batch(model, users, [0] * U)
cand = torch.from_numpy(np.random.default_rng(5).integers(0, cfg.vocab, (U, C)).astype(np.int32)).cuda()
probs = torch.empty((U, C), device="cuda")
for _ in range(3):
    S.score_device(model, cache, cand, probs)
torch.cuda.synchronize()
torch.cuda.profiler.start()
S.score_device(model, cache, cand, probs)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("one scoring call done")
