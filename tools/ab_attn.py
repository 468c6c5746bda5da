"""A/B the tcgen05 cross attention against the SIMT kernels on one config (debug helper)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04421_b200 import ModelConfig, init_params, synthetic_batch  # noqa: E402
from paper_2505_04421_b200.model import LongerModel  # noqa: E402

for kw in [dict(L=64, d=16, K=4, k=16, N=1, m=3), dict(L=256, d=32, K=4, k=32, N=1, m=3),
           dict(L=64, d=16, K=4, k=5, N=1, m=3)]:
    cfg = ModelConfig(**kw).validate()
    P = init_params(cfg, 0)
    rng = np.random.default_rng(1)
    P = {n: a + 0.05 * rng.standard_normal(a.shape) for n, a in P.items()}
    batch = synthetic_batch(cfg, 4, seed=2, min_events=10)
    res = {}
    for flag in ("0", "1"):
        os.environ["LONGER_ATTN_TC"] = flag
        m = LongerModel(cfg)
        m.load_params(P)
        m.loss_backward(batch)
        res[flag] = {n: g.cpu().numpy().copy() for n, g in m.grads()}
        res[flag + "p"] = m._probs[4].cpu().numpy().copy()
    print(kw, "max|dp|", np.abs(res["0p"] - res["1p"]).max())
    for n in ("cross.w_q", "cross.w_k", "cross.w_v", "cross.w_o", "cross.ln1_g", "tables.mlp.seq_w1"):
        a, b = res["0"][n], res["1"][n]
        print(f"  {n}: rel {np.linalg.norm(a - b) / (np.linalg.norm(a) + 1e-30):.3e}")
