import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.params import init_params
from test_parity_gpu import _model
for d, B, me in ((16, 4, 100), (16, 8, 256), (16, 4, 256)):
    cfg = ModelConfig(L=256, d=d, K=4, k=16, N=1, m=3, merge_mode="inner").validate()
    P = init_params(cfg, seed=0)
    batch = synthetic_batch(cfg, B, seed=7, min_events=me)
    ref_p, cache = O.forward(P, cfg, batch.as_dict())
    model = _model(cfg, P)
    X = O.lin(cache["feat"], P["tables.mlp.tok_proj_w"], P["tables.mlp.tok_proj_b"])
    real = cache["real"][:, :, None]
    os.environ["LONGER_DBG_FE"] = "3"
    for rep in range(3):
        p, tr = model.forward_traces(batch)
        H = np.stack([t.h for t in tr])
        err = np.abs(H - X).max(axis=2) / (np.abs(X).max() + 1e-12)
        bad = np.argwhere(~(err < 0.02)).tolist()
        toks = sorted(set(b * 256 + j for b, j in bad))
        tiles = sorted(set(t // 128 for t in toks))
        print(f"d={d} B={B} n_ev>={me} rep{rep}: bad {len(toks)} tiles {tiles} rows", [t % 128 for t in toks][:12], "n_events", batch.n_events.tolist())
