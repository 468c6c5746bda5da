"""Debug: per-group gradient error of the fused / per-stage front-end against a golden file."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_parity_gpu import _golden, _model, _run

path = sys.argv[1]
cfg, P, G, batch, p_ref, loss_ref = _golden(path)
print(cfg.to_dict())
print("dt max", batch.dt.max(), "n_events", batch.n_events)
for fused in ("1", "0"):
    os.environ["LONGER_FUSED"] = fused
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    print(f"fused={fused} max|dp|={np.abs(p - p_ref).max():.2e} loss {loss:.6f} ref {loss_ref:.6f}")
    for name, ref in G.items():
        got = grads[name]
        nr = np.linalg.norm(ref)
        rel = np.linalg.norm(got - ref) / (nr + 1e-30)
        if rel > 0.05:
            print(f"   {name}: rel {rel:.3g} |ref| {nr:.3g} |got| {np.linalg.norm(got):.3g}")
