"""Time inference (longer_forward) and training (longer_forward_backward) at a config with CUDA
events; profiling helper (not the bench).  Usage: python tools/step_probe.py [config] [B]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS  # noqa: E402
from paper_2505_04421_b200 import ModelConfig, synthetic_batch  # noqa: E402
from paper_2505_04421_b200.model import LongerModel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_inner"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
cfg = ModelConfig(**CONFIGS[name]).validate()
model = LongerModel(cfg, seed=0)
batch = synthetic_batch(cfg, B, seed=3).to("cuda")


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


fwd = timed(lambda: model.forward(batch))
train = timed(lambda: model.loss_backward(batch, check=False))
print(f"{name} B={B} fused={os.environ.get('LONGER_FUSED', '1')}: forward {fwd:.3f} ms, "
      f"fwd+bwd {train:.3f} ms")
