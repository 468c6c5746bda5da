"""Stress check of the fused front-end forward: every traced token row (h, merged) of the fused
kernel against the per-stage path, over widths, group sizes, merge modes, batch sizes (tile
counts that leave slots idle / partial tiles) and repeats.  Prints one line per case."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.params import init_params
from paper_2505_04421_b200.model import LongerModel

bad_total = 0
for d, K, merge, L in ((16, 4, "concat", 256), (16, 4, "inner", 256), (32, 4, "concat", 256), (32, 4, "inner", 256),
                       (32, 8, "inner", 512), (32, 2, "inner", 128), (16, 8, "inner", 256), (32, 4, "inner", 2000)):
    cfg = ModelConfig(L=L, d=d, K=K, k=8, N=1, m=3, merge_mode=merge).validate()
    P = init_params(cfg, seed=0)
    rng = np.random.default_rng(1)
    P = {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in P.items()}
    for B in ((1, 3, 8, 37) if L < 2000 else (3, 64)):
        batch = synthetic_batch(cfg, B, seed=B, min_events=1)
        out = {}
        for fused in ("0", "1"):
            os.environ["LONGER_FUSED"] = fused
            m = LongerModel(cfg, seed=0)
            m.load_params(P)
            reps = []
            for _ in range(3 if fused == "1" else 1):
                _, tr = m.forward_traces(batch)
                reps.append((np.stack([t.h for t in tr]), np.stack([t.merged for t in tr])))
            out[fused] = reps
        h0, m0 = out["0"][0]
        bad = 0
        for h1, m1 in out["1"]:
            for a, b in ((h1, h0), (m1, m0)):
                err = np.abs(a - b).max(axis=-1) / (np.abs(b).max() + 1e-12)
                bad += int((~(err < 3e-2)).sum())
        bad_total += bad
        print(f"d={d} K={K} {merge} L={L} B={B}: bad rows {bad}", flush=True)
print("TOTAL BAD", bad_total)
