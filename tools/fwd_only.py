"""Run a few inference forwards at c2 (profiling target for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2505_04421_b200 import ModelConfig, synthetic_batch  # noqa: E402
from paper_2505_04421_b200.model import LongerModel  # noqa: E402

cfg = ModelConfig(**CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2_inner"]).validate()
model = LongerModel(cfg, seed=0)
batch = synthetic_batch(cfg, 256, seed=3).to("cuda")
for _ in range(3):
    model.forward(batch)
torch.cuda.synchronize()
print("ok")
