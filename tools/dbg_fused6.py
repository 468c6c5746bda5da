import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.params import init_params
from test_parity_gpu import _model
d, B = 16, 8
cfg = ModelConfig(L=256, d=d, K=4, k=16, N=1, m=3, merge_mode="inner").validate()
P = init_params(cfg, seed=0)
batch = synthetic_batch(cfg, B, seed=7, min_events=256)
ref_p, cache = O.forward(P, cfg, batch.as_dict())
model = _model(cfg, P)
X = O.lin(cache["feat"], P["tables.mlp.tok_proj_w"], P["tables.mlp.tok_proj_b"])
for dbg in ("3", "5", "6"):
    os.environ["LONGER_DBG_FE"] = dbg
    if dbg in ("5", "6"):
        # modes 5/6 keep the dbg-3 dump through a second flag: dump X too
        pass
    p, tr = model.forward_traces(batch)
    H = np.stack([t.h for t in tr])
    err = np.abs(H - X).max(axis=2) / (np.abs(X).max() + 1e-12)
    bad = np.argwhere(~(err < 0.02)).tolist()
    toks = sorted(set(b * 256 + j for b, j in bad))
    print(f"dbg {dbg}: bad {len(toks)} tiles", sorted(set(t // 128 for t in toks)))
