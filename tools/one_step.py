"""One training step (fwd + bwd + Adam) inside cudaProfilerStart/Stop after warm-up, for
`ncu --profile-from-start off` launch lists.  Usage: python tools/one_step.py [config] [B]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2505_04421_b200 import ModelConfig, synthetic_batch  # noqa: E402
from paper_2505_04421_b200.model import Adam, LongerModel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_inner"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = ModelConfig(**CONFIGS[name]).validate()
model = LongerModel(cfg, seed=0)
opt = Adam(model, cfg.lr)
batch = synthetic_batch(cfg, B, seed=3).to("cuda")
for _ in range(3):
    model.loss_backward(batch, check=False)
    opt.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
model.loss_backward(batch, check=False)
opt.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("one step done")
