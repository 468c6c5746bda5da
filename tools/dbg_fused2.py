import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.params import init_params
from test_parity_gpu import _model, _run, _golden

def check(tag, cfg, P, batch):
    ref_p, cache = O.forward(P, cfg, batch.as_dict())
    extra = cfg.L_padded - cfg.L
    for fused in ("1", "0"):
        os.environ["LONGER_FUSED"] = fused
        model = _model(cfg, P)
        p, tr = model.forward_traces(batch)
        H = np.stack([t.h for t in tr]); Href = cache["h"][:, extra:]
        err = np.abs(H - Href).max(axis=2) / (np.abs(Href).max() + 1e-12)     # [B, L]
        bad = np.argwhere(~(err < 0.05))
        print(tag, "fused", fused, "p err", np.abs(p - ref_p).max(), "bad tokens", len(bad), "of", err.size,
              "first", bad[:8].tolist(), "nan", np.isnan(H).sum())
        if len(bad):
            b, j = bad[0]
            print("   got", H[b, j, :6], "\n   ref", Href[b, j, :6])

for kw in (dict(L=256, d=16, K=4, k=16, N=1, m=3), dict(L=256, d=16, K=4, k=16, N=1, m=3, merge_mode="inner"),
           dict(L=256, d=32, K=4, k=16, N=1, m=3)):
    cfg = ModelConfig(**kw).validate()
    P = init_params(cfg, seed=0)
    check(str(kw), cfg, P, synthetic_batch(cfg, 4, seed=7, min_events=100))
for g in ("small_c1", "small_c2_inner"):
    cfg, P, G, batch, p_ref, loss_ref = _golden(os.path.join(ROOT, "tests/golden", g + ".npz"))
    print(g, cfg.to_dict(), batch.n_events)
    check(g, cfg, P, batch)
