import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.params import init_params
from test_parity_gpu import _model
cfg = ModelConfig(L=256, d=16, K=4, k=16, N=1, m=3).validate()
P = init_params(cfg, seed=0)
batch = synthetic_batch(cfg, 4, seed=7, min_events=100)
ref_p, cache = O.forward(P, cfg, batch.as_dict())
for slots in ("2", "3", "0"):
    os.environ["LONGER_DBG_SLOTS"] = slots
    model = _model(cfg, P)
    for rep in range(2):
        p, tr = model.forward_traces(batch)
        H = np.stack([t.h for t in tr]); Href = cache["h"]
        err = np.abs(H - Href).max(axis=2) / (np.abs(Href).max() + 1e-12)
        print("slots", slots, "rep", rep, "bad", int((~(err < 0.05)).sum()), H[0, 70, :4], Href[0, 70, :4])
