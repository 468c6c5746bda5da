import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04421_b200 import ModelConfig, init_params, synthetic_batch
from paper_2505_04421_b200.model import LongerModel
from oracle import longer_oracle as O
kw = dict(L=256, d=32, K=4, k=32, N=1, m=3)
cfg = ModelConfig(**kw).validate()
P = init_params(cfg, 0)
rng = np.random.default_rng(1)
P = {n: a + 0.05 * rng.standard_normal(a.shape) for n, a in P.items()}
batch = synthetic_batch(cfg, 4, seed=2, min_events=10)
print("n_events", batch.n_events)
p_ref, loss_ref, _ = O.forward_backward(P, cfg, batch.as_dict())
print("oracle p", p_ref, loss_ref)
for fused in ("0", "1"):
    for tc in ("0", "1"):
        os.environ["LONGER_FUSED"] = fused; os.environ["LONGER_ATTN_TC"] = tc
        m = LongerModel(cfg); m.load_params(P)
        try:
            l = m.loss_backward(batch)
        except Exception as e:
            l = repr(e)
        print(fused, tc, "loss", l, "p", m._probs[4].cpu().numpy(), "fwd", m.forward(batch).cpu().numpy())
