"""Parity of the sm_100a path (through the C ABI) with the reference.

* golden vectors produced by the reference itself (tests/golden/*.npz, d % 8 == 0 cases);
* the float64 oracle on seeded synthetic batches, including the c2 shape (L=2000, d=32, K=4,
  k=32, N=2, InnerTrans) at a batch the oracle finishes in seconds.

Stated tolerance (bf16 operands, fp32 accumulation / softmax / LN):
  |Δp| ≤ 5e-3 per sample;
  |Δloss| ≤ mean_b 5e-3·|dBCE/dp|_b + 1e-4 (the loss error the per-sample p tolerance allows);
  per-parameter gradient: rel-L2 ≤ 0.15 and cosine ≥ 0.995 when ‖g‖ is not negligible
  (every backward GEMM also takes bf16 operands, so gradients carry two roundings per layer);
  groups whose exact gradient is ~0 (every b_k: softmax shift invariance) must be ≤ 1e-3·max‖g‖.
"""
import glob
import json
import os

import numpy as np
import pytest

from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.inputs import Batch

pytestmark = pytest.mark.gpu

GOLDEN = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                if not os.path.basename(p).startswith("serving_"))


def _golden(path):
    z = np.load(path)
    cfg = ModelConfig(**json.loads(str(z["cfg"])))
    P = {k[2:]: z[k] for k in z.files if k.startswith("P/")}
    G = {k[2:]: z[k] for k in z.files if k.startswith("G/")}
    batch = Batch(**{k[6:]: z[k] for k in z.files if k.startswith("batch/")})
    return cfg, P, G, batch, z["p"], float(z["loss"])


def _model(cfg, P):
    from paper_2505_04421_b200.model import LongerModel
    m = LongerModel(cfg, seed=0)
    m.load_params(P)
    return m


def assert_grads_close(grads_dev, G, tag=""):
    scale = max(float(np.linalg.norm(g)) for g in G.values())
    bad = []
    for name, ref in G.items():
        got = grads_dev[name]
        nr = float(np.linalg.norm(ref))
        diff = float(np.linalg.norm(got - ref))
        if nr <= 1e-3 * scale:
            if diff > 1e-3 * scale + 1e-7:
                bad.append(f"{name}: |g|~0 ref, diff {diff:.3g} (scale {scale:.3g})")
            continue
        cos = float(np.dot(got.ravel(), ref.ravel()) / (np.linalg.norm(got) * nr + 1e-30))
        if diff / nr > 0.15 or cos < 0.995:
            bad.append(f"{name}: rel {diff / nr:.3g} cos {cos:.5f}")
    assert not bad, tag + "\n" + "\n".join(bad)


def loss_tol(p_ref, labels):
    p = np.clip(p_ref, 1e-12, 1 - 1e-12)
    y = np.asarray(labels, dtype=np.float64)
    return float(np.mean(5e-3 * np.abs(y / p - (1 - y) / (1 - p)))) + 1e-4


def _run(model, batch):
    loss = model.loss_backward(batch)
    p = model._probs[batch.size].cpu().numpy().astype(np.float64)
    grads = {n: g.detach().cpu().numpy().astype(np.float64) for n, g in model.grads()}
    return p, loss, grads


DEVICE_GOLDEN = [p for p in GOLDEN if json.loads(str(np.load(p)["cfg"]))["d"] % 8 == 0]


@pytest.mark.parametrize("path", DEVICE_GOLDEN, ids=[os.path.basename(p)[:-4] for p in DEVICE_GOLDEN])
def test_forward_backward_matches_reference_golden(path):
    cfg, P, G, batch, p_ref, loss_ref = _golden(path)
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    assert np.max(np.abs(p - p_ref)) <= 5e-3, np.abs(p - p_ref)
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label), (loss, loss_ref)
    assert_grads_close(grads, G, os.path.basename(path))
    # inference entry point agrees with the training forward
    p2 = model.forward(batch).cpu().numpy()
    np.testing.assert_allclose(p2, p, rtol=0, atol=2e-3)   # fused vs unfused front-end


C2 = dict(L=2000, d=32, K=4, k=32, N=2, m=3, merge_mode="inner")


@pytest.mark.parametrize("kw,B,min_events", [
    (C2, 3, None),
    (dict(C2, merge_mode="concat"), 3, None),
    (dict(C2, L=512), 4, 1),
    (dict(L=256, d=16, K=4, k=16, N=1, m=3), 8, 100),
    # c5 widths (D = 256, K = 8): per-stage MLP backward fallback, head width 256 (SIMT attention)
    (dict(L=96, d=32, K=8, k=4, N=2, m=3, merge_mode="inner"), 3, 20),
    # the other query strategies at the c2 widths, mixed lengths (pad queries included)
    (dict(C2, L=512, query_strategy="uniform"), 4, 1),
    (dict(C2, L=512, query_strategy="recent_uniform", merge_mode="concat"), 4, 1),
    (dict(C2, L=512, query_strategy="learnable"), 4, 1),
    # D = 256 with two heads: tensor-core attention at head width 128
    (dict(L=96, d=32, K=8, k=4, N=1, m=3, heads=2, merge_mode="inner"), 3, 20),
    # the other fused front-end instantiations: token width 32 with K = 2 (D = 64) and token width
    # 16 with K = 8 (D = 128), InnerTrans and concat, ragged lengths
    (dict(L=300, d=32, K=2, k=8, N=1, m=3, merge_mode="inner"), 4, 50),
    (dict(L=300, d=16, K=8, k=8, N=1, m=3, merge_mode="inner"), 4, 50),
    (dict(L=300, d=16, K=8, k=8, N=2, m=3, merge_mode="concat"), 4, 50),
])
def test_matches_oracle_on_synthetic(kw, B, min_events):
    cfg = ModelConfig(**kw).validate()
    from paper_2505_04421_b200.params import init_params
    P = init_params(cfg, seed=0)
    # perturb the structured init so that every gradient path is exercised
    rng = np.random.default_rng(3)
    P = {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in P.items()}
    batch = synthetic_batch(cfg, B, seed=7, min_events=min_events)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    assert np.max(np.abs(p - p_ref)) <= 5e-3
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label)
    assert_grads_close(grads, G, str(kw))
    # inference entry point (fused front-end when the shape allows it)
    pf = model.forward(batch).cpu().numpy().astype(np.float64)
    assert np.max(np.abs(pf - p_ref)) <= 5e-3, np.abs(pf - p_ref)


@pytest.mark.parametrize("pack,tma", [("0", "1"), ("2", "1"), ("2", "0"), ("1", "0")])
def test_attention_variants_match_oracle(pack, tma, monkeypatch):
    """Every tensor-core attention variant (read per launch): samples packed per CTA in the
    self layers (LONGER_ATTN_PACK: 0 off, 1 backward only = default, 2 forward too) x K/V by TMA or
    by thread loads (LONGER_ATTN_TMA), at the c2 widths with mixed lengths, a query strategy that
    gathers query groups, and B = 4 (a partly filled packed CTA)."""
    monkeypatch.setenv("LONGER_ATTN_PACK", pack)
    monkeypatch.setenv("LONGER_ATTN_TMA", tma)
    cfg = ModelConfig(**dict(C2, L=512, query_strategy="uniform")).validate()
    from paper_2505_04421_b200.params import init_params
    P = init_params(cfg, seed=0)
    rng = np.random.default_rng(5)
    P = {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in P.items()}
    batch = synthetic_batch(cfg, 4, seed=11, min_events=1)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    assert np.max(np.abs(p - p_ref)) <= 5e-3
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label)
    assert_grads_close(grads, G, f"pack={pack} tma={tma}")


def test_kv_layernorm_backward_matches_oracle():
    """The K/V-row LayerNorm backward (half-warp rows through a cp.async ring) matches the oracle
    with mixed lengths and B = 5, so the last ring stage holds a partial group of rows."""
    cfg = ModelConfig(**dict(C2, L=512)).validate()
    from paper_2505_04421_b200.params import init_params
    P = init_params(cfg, seed=0)
    rng = np.random.default_rng(9)
    P = {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in P.items()}
    batch = synthetic_batch(cfg, 5, seed=23, min_events=1)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    assert np.max(np.abs(p - p_ref)) <= 5e-3
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label)
    assert_grads_close(grads, G, "kv ln backward")


@pytest.mark.parametrize("head_rows", ["1", "0"])
def test_last_block_head_rows_match_oracle(head_rows, monkeypatch):
    """The last self block's row-wise tail on the two head rows only (default) and on all rows
    (LONGER_HEAD_ROWS=0) both match the oracle, forward and backward, at N = 1 and N = 2."""
    monkeypatch.setenv("LONGER_HEAD_ROWS", head_rows)
    for kw in (dict(C2, L=512), dict(C2, L=512, N=1, m=4)):
        cfg = ModelConfig(**kw).validate()
        from paper_2505_04421_b200.params import init_params
        P = init_params(cfg, seed=0)
        rng = np.random.default_rng(8)
        P = {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in P.items()}
        batch = synthetic_batch(cfg, 5, seed=17, min_events=1)
        p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
        model = _model(cfg, P)
        p, loss, grads = _run(model, batch)
        assert np.max(np.abs(p - p_ref)) <= 5e-3
        assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label)
        assert_grads_close(grads, G, f"head_rows={head_rows} {kw}")
        pf = model.forward(batch).cpu().numpy().astype(np.float64)
        assert np.max(np.abs(pf - p_ref)) <= 5e-3


@pytest.mark.parametrize("bias", [20.0, 40.0, -40.0, -25.0])
def test_saturated_logits_follow_the_reference_clamp(bias):
    """p = sigmoid(z) saturates in fp32 long before the reference's 1e-12 clamp does; the loss and
    the clamp's zero-gradient region must still follow tensors.py:551-571 (float64)."""
    cfg = ModelConfig(L=48, d=8, K=2, k=6, N=1, n_users=40).validate()
    from paper_2505_04421_b200.params import init_params
    P = init_params(cfg, seed=0)
    P["head.b2"] = P["head.b2"] + bias
    batch = synthetic_batch(cfg, 4, seed=3)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    assert np.isfinite(loss)
    assert abs(loss - loss_ref) <= 1e-3 * abs(loss_ref) + 1e-3, (loss, loss_ref)
    assert_grads_close(grads, {n: G[n] for n in ("head.b2", "head.w2", "head.w1", "cross.w_v", "tables.item_table")},
                       f"bias {bias}")


def test_autograd_bridge_matches_training_step():
    """torch.autograd path (LongerFunction → longer_backward VJP) ≡ the fused training step for the
    same BCE loss away from the clamp region, and against the oracle."""
    import torch
    cfg = ModelConfig(L=256, d=16, K=4, k=16, N=1, m=3).validate()
    from paper_2505_04421_b200.params import init_params
    rng = np.random.default_rng(11)
    P = {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in init_params(cfg, seed=0).items()}
    batch = synthetic_batch(cfg, 6, seed=5, min_events=60)
    model = _model(cfg, P)
    _, _, G_step = _run(model, batch)
    probs = model.probs(batch)
    y = torch.from_numpy(np.asarray(batch.label)).cuda()
    loss = torch.nn.functional.binary_cross_entropy(probs, y)
    loss.backward()
    flat = model.autograd_params().grad.detach().cpu().numpy().astype(np.float64)
    off = 0
    G_ag = {}
    for name, shape in model.shapes.items():
        n = int(np.prod(shape))
        G_ag[name] = flat[off:off + n].reshape(shape)
        off += n
    for name in G_step:
        np.testing.assert_allclose(G_ag[name], G_step[name], rtol=2e-3, atol=1e-6, err_msg=name)
    _, _, G_ref = O.forward_backward(P, cfg, batch.as_dict())
    assert_grads_close(G_ag, G_ref, "autograd")
    # a second forward invalidates the first one's saved activations
    p1 = model.probs(batch)
    model.forward(batch)
    with pytest.raises(RuntimeError):
        p1.sum().backward()
