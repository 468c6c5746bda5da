import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.params import init_params
from test_parity_gpu import _model
for d in (16, 32):
    cfg = ModelConfig(L=256, d=d, K=4, k=16, N=1, m=3, merge_mode="inner").validate()
    P = init_params(cfg, seed=0)
    batch = synthetic_batch(cfg, 4, seed=7, min_events=100)
    ref_p, cache = O.forward(P, cfg, batch.as_dict())
    model = _model(cfg, P)
    X = O.lin(cache["feat"], P["tables.mlp.tok_proj_w"], P["tables.mlp.tok_proj_b"])
    POS = P["tables.abs_pos_table"][cache["rec"]]
    real = cache["real"][:, :, None]
    for dbg, R in (("3", X * real), ("4", POS * real)):
        os.environ["LONGER_DBG_FE"] = dbg
        p, tr = model.forward_traces(batch)
        H = np.stack([t.h for t in tr]) * real
        err = np.abs(H - R).max(axis=2) / (np.abs(R).max() + 1e-12)
        bad = np.argwhere(~(err < 0.02))
        print("d", d, dbg, "bad", len(bad), bad[:5].tolist(), "\n  got", H[0, 70, :6], "\n  ref", R[0, 70, :6])
