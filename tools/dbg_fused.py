"""Debug: fused vs per-stage vs oracle on synthetic batches (no golden)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.params import init_params
from test_parity_gpu import _model, _run

for kw in (dict(L=256, d=16, K=4, k=16, N=1, m=3), dict(L=256, d=32, K=4, k=16, N=2, m=3, merge_mode="inner")):
    cfg = ModelConfig(**kw).validate()
    P = init_params(cfg, seed=0)
    rng = np.random.default_rng(3)
    P = {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in P.items()}
    batch = synthetic_batch(cfg, 4, seed=7, min_events=100)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    for fused in ("1", "0"):
        os.environ["LONGER_FUSED"] = fused
        model = _model(cfg, P)
        pf = model.forward(batch).cpu().numpy()
        print(kw, f"fused={fused} forward max|dp|={np.abs(pf - p_ref).max():.2e}", np.isnan(pf).sum())
        _, tr = model.forward_traces(batch)
        ref_p, cache = O.forward(P, cfg, batch.as_dict())
        extra = cfg.L_padded - cfg.L
        for i, t in enumerate(tr[:1]):
            for nm, got, ref in (("h", t.h, cache["h"][i, extra:]), ("merged", t.merged, cache["merged"][i])):
                err = np.abs(got - ref).max() / (np.abs(ref).max() + 1e-12)
                print(f"   {nm}: rel max err {err:.3e} nan {np.isnan(got).sum()}")
        try:
            p, loss, grads = _run(model, batch)
        except Exception as exc:
            print("   step failed:", exc)
            continue
        print(f"   step max|dp|={np.abs(p - p_ref).max():.2e} loss {loss:.6f} ref {loss_ref:.6f}")
        scale = max(np.linalg.norm(g) for g in G.values())
        for name, ref in G.items():
            nr = np.linalg.norm(ref)
            rel = np.linalg.norm(grads[name] - ref) / (nr + 1e-30)
            if rel > 0.05 and nr > 1e-3 * scale:
                print(f"   {name}: rel {rel:.3g} |ref| {nr:.3g} |got| {np.linalg.norm(grads[name]):.3g}")
