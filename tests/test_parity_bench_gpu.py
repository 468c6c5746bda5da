"""Parity at the benchmarked configuration, and in the kernels' multi-tile modes.

`bench.py` times the train-step body (pkg/src/longrec/model.py:555-567) at c2 with B = 256 per
GPU.  At that batch every fused front-end CTA walks many 128-token tiles and accumulates its
weight gradients (token MLP, featuriser one-hots, InnerTrans layer) in TMEM across them, and the
row-level GEMMs take their 128/256-wide fused-epilogue tiles.  These tests run exactly that call
(`LongerModel.loss_backward`, through the C ABI) against the float64 oracle:

* c2-inner and c2-concat at B = 256 — the bench batch itself, with full-length and with mixed
  lengths; the oracle runs in chunks of 32 samples and the batch gradient is the size-weighted
  mean of the chunk gradients (the loss is a batch mean, model.py:558-562);
* a small batch with the fused grids capped (LONGER_FE_GRID) so that each CTA takes ≥ 8 tiles,
  and LONGER_GEMM_MIN_TILES=1 so every GEMM takes its widest tile and fused epilogue.

Stated tolerance: as tests/test_parity_gpu.py (|Δp| ≤ 5e-3; loss within the BCE slope of that;
per-group gradients rel-L2 ≤ 0.15 and cosine ≥ 0.995, ~0 groups absolute).
"""
import numpy as np
import pytest

from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.params import init_params

from test_parity_gpu import _model, _run, assert_grads_close, loss_tol

pytestmark = pytest.mark.gpu

C2 = dict(L=2000, d=32, K=4, k=32, N=2, m=3, merge_mode="inner")


def oracle_chunked(P, cfg, batch, chunk=32):
    """p, mean loss and mean gradients of the whole batch, from float64 oracle chunks."""
    B = batch.size
    d = batch.as_dict()
    ps, loss, G = [], 0.0, None
    for lo in range(0, B, chunk):
        sub = {k: v[lo:lo + chunk] for k, v in d.items()}
        n = len(sub["label"])
        p, l, g = O.forward_backward(P, cfg, sub)
        ps.append(p)
        loss += l * n
        if G is None:
            G = {k: v * n for k, v in g.items()}
        else:
            for k, v in g.items():
                G[k] += v * n
    return np.concatenate(ps), loss / B, {k: v / B for k, v in G.items()}


def _perturbed(cfg, seed):
    rng = np.random.default_rng(seed)
    return {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in init_params(cfg, seed=0).items()}


@pytest.mark.parametrize("merge,min_events", [("inner", None), ("concat", None), ("inner", 1)],
                         ids=["c2-inner", "c2-concat", "c2-inner-mixed"])
def test_bench_batch_matches_oracle(merge, min_events):
    cfg = ModelConfig(**dict(C2, merge_mode=merge)).validate()
    P = _perturbed(cfg, 21)
    batch = synthetic_batch(cfg, 256, seed=1, min_events=min_events)
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    p_ref, loss_ref, G = oracle_chunked(P, cfg, batch)
    dp = np.abs(p - p_ref)
    assert dp.max() <= 5e-3, (dp.max(), int(dp.argmax()))
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label), (loss, loss_ref)
    assert_grads_close(grads, G, f"B=256 {merge} min_events={min_events}")


@pytest.mark.parametrize("fe_split", ["0", "2"], ids=["column-blocks", "split-ranges"])
@pytest.mark.parametrize("merge", ["inner", "concat"])
def test_multi_tile_per_cta_matches_oracle(merge, fe_split, monkeypatch):
    """Fused grids capped at 3 CTAs (fe_fwd / fe_inner_bwd: ~30 tiles each; fe_mlp_bwd: one CTA
    per 128-token column block, each walking every sample — or, split, 3 CTAs each walking a third
    of the column-block-major tile order across column-block changes), every GEMM at its widest tile."""
    monkeypatch.setenv("LONGER_FE_GRID", "3")
    monkeypatch.setenv("LONGER_FE_SPLIT", fe_split)
    monkeypatch.setenv("LONGER_GEMM_MIN_TILES", "1")
    cfg = ModelConfig(**dict(C2, merge_mode=merge)).validate()
    P = _perturbed(cfg, 13)
    batch = synthetic_batch(cfg, 10, seed=5, min_events=1)
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    assert np.max(np.abs(p - p_ref)) <= 5e-3
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label)
    assert_grads_close(grads, G, f"capped grid {merge}")
    # the capped and the full grids compute the same step (fp32 accumulation order aside)
    monkeypatch.delenv("LONGER_FE_GRID")
    monkeypatch.delenv("LONGER_GEMM_MIN_TILES")
    monkeypatch.delenv("LONGER_FE_SPLIT")
    p2, loss2, grads2 = _run(model, batch)
    np.testing.assert_allclose(p2, p, atol=1e-4)
    for name in grads:
        scale = np.abs(grads[name]).max() + 1e-12
        assert np.abs(grads2[name] - grads[name]).max() <= 2e-3 * scale + 1e-7, name


C5 = dict(L=10000, d=32, K=8, k=32, N=4, m=3, merge_mode="inner")


@pytest.mark.parametrize("min_events,fe_split", [(None, "1"), (3000, "1"), (3000, "2")],
                         ids=["full", "mixed", "mixed-split"])
def test_c5_real_shape_matches_oracle(min_events, fe_split, monkeypatch):
    """BASELINE config 5 at its real shape (L = 10,000, d = 32, K = 8 → D = 256, N = 4 self
    layers, InnerTrans): 1,250 merged keys = 10 key chunks of the tensor-core attention at head
    width 256, the fused forward at D = 256 (three tile slots per CTA), the 256-wide K/V-row LN
    backward, and the fused token-MLP backward in two passes of 256 hidden units (2D = 512) with the
    partial dx0 handed between them — in column-block mode, and (mixed-split) in the split mode the
    bench's B = 256 runs, where each CTA's tile range crosses column blocks."""
    monkeypatch.setenv("LONGER_FE_SPLIT", fe_split)
    cfg = ModelConfig(**C5).validate()
    P = _perturbed(cfg, 31)
    batch = synthetic_batch(cfg, 4, seed=2, min_events=min_events)
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    p_ref, loss_ref, G = oracle_chunked(P, cfg, batch, chunk=2)
    assert np.max(np.abs(p - p_ref)) <= 5e-3, np.abs(p - p_ref)
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label), (loss, loss_ref)
    assert_grads_close(grads, G, f"c5 min_events={min_events}")
    pf = model.forward(batch).cpu().numpy().astype(np.float64)
    assert np.max(np.abs(pf - p_ref)) <= 5e-3


@pytest.mark.parametrize("heads", [1, 2], ids=["dh128", "dh64"])
def test_cross_attention_backward_double_buffered_path(heads, monkeypatch):
    """The cross layer's attention backward (35 queries, 503 keys = 4 chunks, one sample per CTA)
    runs the SHORT variant: 64-row query tiles, two K / V buffers with the TMA of chunk i+2 in
    flight, staged dV / dK stores.  Same oracle bar as above, and the same step as the
    single-buffer variant (LONGER_ATTN_SHORT=0) up to fp32 accumulation order."""
    cfg = ModelConfig(**dict(C2, heads=heads)).validate()
    P = _perturbed(cfg, 17)
    batch = synthetic_batch(cfg, 6, seed=9, min_events=1)
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    assert np.max(np.abs(p - p_ref)) <= 5e-3
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label)
    assert_grads_close(grads, G, f"cross bwd short heads={heads}")
    monkeypatch.setenv("LONGER_ATTN_SHORT", "0")
    p2, loss2, grads2 = _run(model, batch)
    np.testing.assert_allclose(p2, p, atol=1e-6)
    top = max(np.abs(g).max() for g in grads.values())
    for name in grads:                    # ~0 groups (e.g. b_k: softmax-invariant) are rounding noise
        scale = max(np.abs(grads[name]).max(), 1e-2 * top)
        assert np.abs(grads2[name] - grads[name]).max() <= 1e-3 * scale, name


@pytest.mark.parametrize("merge", ["inner", "concat"])
def test_absorbed_cross_kv_projections(merge, monkeypatch):
    """Cross layer with the K/V projections absorbed (heads = 1, the default): scores Q'·knᵀ with
    Q' = Q·W_kᵀ, context (P·kn)·W_v + b_v, no [K | V] rows over the B·v key rows; backward through
    dC = dctx·W_vᵀ, d(kn) = dK + dV from one attention pass, dQ = dQ'·W_k, dW_k = dQ'ᵀ·Q.  Both
    the absorbed and the explicit path (LONGER_ABSORB_KV=0) meet the oracle bar; the absorbed
    cross.b_k gradient is exactly 0 (the softmax is invariant to b_k; the reference's is rounding
    noise around 0)."""
    cfg = ModelConfig(**dict(C2, merge_mode=merge)).validate()
    P = _perturbed(cfg, 23)
    batch = synthetic_batch(cfg, 6, seed=4, min_events=1)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    model = _model(cfg, P)
    for absorb in ("1", "0"):
        monkeypatch.setenv("LONGER_ABSORB_KV", absorb)
        p, loss, grads = _run(model, batch)
        assert np.max(np.abs(p - p_ref)) <= 5e-3, absorb
        assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label), absorb
        assert_grads_close(grads, G, f"absorb={absorb} {merge}")
        if absorb == "1":
            assert not np.any(grads["cross.b_k"])
            pf = model.forward(batch).cpu().numpy().astype(np.float64)
            assert np.max(np.abs(pf - p_ref)) <= 5e-3


def test_shared_kv_tile_matches_separate_tiles(monkeypatch):
    """With absorbed projections the cross attention's keys and values are the same rows: one TMA
    tile per chunk serves both (and dV + dK accumulate in one TMEM region).  Same step as loading
    the rows twice (LONGER_ATTN_KVS=0) up to fp32 accumulation order."""
    cfg = ModelConfig(**C2).validate()
    P = _perturbed(cfg, 29)
    batch = synthetic_batch(cfg, 6, seed=8, min_events=1)
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    monkeypatch.setenv("LONGER_ATTN_KVS", "0")
    p2, loss2, grads2 = _run(model, batch)
    np.testing.assert_allclose(p2, p, atol=1e-6)
    top = max(np.abs(g).max() for g in grads.values())
    for name in grads:
        scale = max(np.abs(grads[name]).max(), 1e-2 * top)
        assert np.abs(grads2[name] - grads[name]).max() <= 1e-3 * scale, name


@pytest.mark.parametrize("heads_D", [(1, 128), (1, 64)], ids=["D128", "D64"])
def test_keys_as_rows_cross_attention_backward(heads_D, monkeypatch):
    """The absorbed cross layer's attention backward with the keys as the tile rows (Sᵀ / dPᵀ
    double-buffered in TMEM, every worker lane a key row): the oracle bar, and the same step as
    the query-row kernel (LONGER_ATTN_BWD_T=0) up to fp32 accumulation order."""
    heads, D = heads_D
    cfg = ModelConfig(**dict(C2, d=D // 4, heads=heads)).validate()
    P = _perturbed(cfg, 37)
    batch = synthetic_batch(cfg, 6, seed=12, min_events=1)
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    assert np.max(np.abs(p - p_ref)) <= 5e-3
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label)
    assert_grads_close(grads, G, f"bwd_t D={D}")
    monkeypatch.setenv("LONGER_ATTN_BWD_T", "0")
    p2, loss2, grads2 = _run(model, batch)
    np.testing.assert_allclose(p2, p, atol=1e-6)
    top = max(np.abs(g).max() for g in grads.values())
    for name in grads:
        scale = max(np.abs(grads[name]).max(), 1e-2 * top)
        assert np.abs(grads2[name] - grads[name]).max() <= 2e-3 * scale, name


@pytest.mark.parametrize("fe_grid", [None, "3"], ids=["full-grid", "capped-grid"])
def test_d16_inner_trans_fused_backward(fe_grid, monkeypatch):
    """Token width 16 with InnerTrans (D = 64, FFN hidden 4d = 64 < 128): the fused InnerTrans
    backward's weight-gradient MMAs take the hidden units as their M = 128 dimension, so the
    64-wide FFN tiles are padded to 128-element rows and only accumulator rows < 64 are flushed
    (found by this test: before, rows 64-127 were misread and added past W2's gradient)."""
    if fe_grid:
        monkeypatch.setenv("LONGER_FE_GRID", fe_grid)
    cfg = ModelConfig(**dict(C2, d=16)).validate()
    P = _perturbed(cfg, 37)
    batch = synthetic_batch(cfg, 6, seed=12, min_events=1)
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    p_ref, loss_ref, G = O.forward_backward(P, cfg, batch.as_dict())
    assert np.max(np.abs(p - p_ref)) <= 5e-3
    assert abs(loss - loss_ref) <= loss_tol(p_ref, batch.label)
    assert_grads_close(grads, G, f"d16 inner fe_grid={fe_grid}")


def test_pdl_fences_do_not_change_the_step(monkeypatch):
    """LONGER_PDL_FENCE only changes which launches may start early (scheduling): the step with
    every fence, with none and with PDL off computes the same probabilities and gradients (fp32
    atomic accumulation order aside)."""
    cfg = ModelConfig(**C2).validate()
    P = _perturbed(cfg, 23)
    batch = synthetic_batch(cfg, 12, seed=4, min_events=1)
    model = _model(cfg, P)
    p, loss, grads = _run(model, batch)
    for env in [("LONGER_PDL_FENCE", "0"), ("LONGER_PDL_FENCE", "255"), ("LONGER_PDL", "0")]:
        monkeypatch.setenv(*env)
        p2, loss2, grads2 = _run(model, batch)
        monkeypatch.delenv(env[0])
        np.testing.assert_allclose(p2, p, atol=1e-6)
        for name in grads:
            scale = np.abs(grads[name]).max() + 1e-12
            assert np.abs(grads2[name] - grads[name]).max() <= 1e-4 * scale + 1e-9, (env, name)
