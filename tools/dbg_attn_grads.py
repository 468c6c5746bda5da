"""Per-group gradient error vs the oracle at the reference init (the bench's weights), c2 shape."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.params import init_params
from test_parity_gpu import _model, _run
for kw in (dict(L=2000, d=32, K=4, k=32, N=2, m=3, merge_mode="inner"), dict(L=256, d=16, K=4, k=16, N=1, m=3)):
    cfg = ModelConfig(**kw).validate()
    P = init_params(cfg, seed=0)
    batch = synthetic_batch(cfg, 6, seed=3, min_events=50)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    scale = max(np.linalg.norm(g) for g in G.values())
    out = []
    for n in ("cross.w_q", "cross.w_k", "cross.w_v", "self.0.w_q", "self.0.w_k", "tables.mlp.seq_w1"):
        if n not in G: continue
        nr = np.linalg.norm(G[n]); rel = np.linalg.norm(grads[n] - G[n]) / (nr + 1e-30)
        out.append(f"{n}: rel {rel:.3f} |g|/scale {nr/scale:.1e}")
    print(kw["L"], f"dp {np.abs(p - p_ref).max():.1e}", "; ".join(out))
