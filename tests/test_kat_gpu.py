"""Known-answer and invariance tests of the reference, ported to the sm_100a path.

* zero head → p = 0.5 exactly (pkg/tests/test_model.py:92-97);
* masked inputs are exactly ignored: events outside a sample's last n_events (the left padding)
  never reach a visible key, so rewriting them leaves p bit-identical (the spirit of
  pkg/tests/test_tensors.py:129-138 and the prefix/target-row invariances of
  pkg/tests/test_attention.py:216-250); the candidate does reach p (test_model.py:100-109);
* samples are independent: p of a sample does not depend on the rest of the batch (bit-identical);
* very short histories (every sequence query a pad query → fully masked attention rows, whose
  context is exactly 0, pkg/tests/test_tensors.py:110-112) match the oracle;
* the fused Adam step follows Adam.step (pkg/src/longrec/model.py:467-482).
"""
import numpy as np
import pytest

from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.inputs import Batch

pytestmark = pytest.mark.gpu

C2 = dict(L=2000, d=32, K=4, k=32, N=2, m=3, merge_mode="inner")


def _model(cfg, P=None):
    from paper_2505_04421_b200.model import LongerModel
    m = LongerModel(cfg, seed=0)
    if P is not None:
        m.load_params(P)
    return m


def _copy(b: Batch, **over) -> Batch:
    d = {f: np.array(getattr(b, f), copy=True) for f in Batch.FIELDS}
    d.update(over)
    return Batch(**d)


def test_zero_head_gives_half_exactly():
    cfg = ModelConfig(**dict(C2, L=512)).validate()
    from paper_2505_04421_b200.params import init_params
    P = init_params(cfg, seed=0)
    P["head.w2"] = np.zeros_like(P["head.w2"])
    P["head.b2"] = np.zeros_like(P["head.b2"])
    p = _model(cfg, P).forward(synthetic_batch(cfg, 8, seed=3, min_events=1)).cpu().numpy()
    assert np.all(p == 0.5), p


@pytest.mark.parametrize("merge_mode", ["inner", "concat"])
def test_padding_events_are_exactly_ignored(merge_mode):
    cfg = ModelConfig(**dict(C2, L=512, merge_mode=merge_mode)).validate()
    model = _model(cfg)
    b = synthetic_batch(cfg, 6, seed=5, min_events=1)
    rng = np.random.default_rng(9)
    pad = np.arange(cfg.L)[None, :] < (cfg.L - b.n_events)[:, None]
    noisy = _copy(b,
                  items=np.where(pad, rng.integers(0, cfg.vocab, b.items.shape), b.items).astype(np.int32),
                  actions=np.where(pad, rng.integers(0, cfg.n_actions, b.actions.shape), b.actions).astype(np.int32),
                  dt=np.where(pad, rng.integers(1, 10**6, b.dt.shape), b.dt).astype(np.int32))
    assert (noisy.items != b.items).any()
    p0 = model.forward(b).cpu().numpy()
    p1 = model.forward(noisy).cpu().numpy()
    np.testing.assert_array_equal(p0, p1)
    # the candidate, in contrast, reaches p
    other = _copy(b, cand_item=((b.cand_item + 1) % cfg.vocab).astype(np.int32))
    assert np.all(model.forward(other).cpu().numpy() != p0)


def test_samples_are_independent_of_the_rest_of_the_batch():
    cfg = ModelConfig(**C2).validate()
    model = _model(cfg)
    a = synthetic_batch(cfg, 12, seed=21, min_events=100)
    b = synthetic_batch(cfg, 12, seed=22, min_events=100)
    # batch c = the first 5 samples of a followed by 7 samples of b
    mixed = Batch(**{f: np.concatenate([getattr(a, f)[:5], getattr(b, f)[5:]]) for f in Batch.FIELDS})
    pa = model.forward(a).cpu().numpy()
    pm = model.forward(mixed).cpu().numpy()
    np.testing.assert_array_equal(pa[:5], pm[:5])
    # and alone (a different batch size: other tile shapes, other grid)
    p1 = model.forward(Batch(**{f: getattr(a, f)[2:3] for f in Batch.FIELDS})).cpu().numpy()
    np.testing.assert_array_equal(pa[2:3], p1)


@pytest.mark.parametrize("n_events", [1, 3, 4, 9])
def test_short_histories_match_oracle(n_events):
    """n_events < K·k: most (n = 1, 3: all but one or all) sequence queries are pad queries whose
    attention rows are fully masked."""
    cfg = ModelConfig(**dict(C2, L=256)).validate()
    from paper_2505_04421_b200.params import init_params
    P = init_params(cfg, seed=0)
    rng = np.random.default_rng(4)
    P = {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in P.items()}
    b = synthetic_batch(cfg, 3, seed=13)
    real = np.arange(cfg.L)[None, :] >= cfg.L - n_events
    b = _copy(b, n_events=np.full(3, n_events, np.int32),
              items=np.where(real, b.items, 0).astype(np.int32),
              actions=np.where(real, b.actions, 0).astype(np.int32),
              dt=np.where(real, b.dt, 0).astype(np.int32))
    p_ref, loss_ref, G = O.forward_backward(P, cfg, b.as_dict())
    model = _model(cfg, P)
    loss = model.loss_backward(b)
    p = model._probs[b.size].cpu().numpy().astype(np.float64)
    assert np.max(np.abs(p - p_ref)) <= 5e-3
    grads = {n: g.detach().cpu().numpy().astype(np.float64) for n, g in model.grads()}
    from test_parity_gpu import assert_grads_close, loss_tol
    assert abs(loss - loss_ref) <= loss_tol(p_ref, b.label)
    assert_grads_close(grads, G, f"n_events={n_events}")


def test_adam_matches_reference_update():
    """longer_adam_step against Adam.step of the reference (model.py:467-482, restated as
    oracle.adam_step) over several steps with changing gradients; fp32 state vs float64."""
    import torch
    from paper_2505_04421_b200.model import Adam
    cfg = ModelConfig(**dict(C2, L=256)).validate()
    model = _model(cfg)
    rng = np.random.default_rng(2)
    n = model.flat.numel()
    p_ref = rng.standard_normal(n) * 0.1
    m_ref, v_ref = np.zeros(n), np.zeros(n)
    model.flat.copy_(torch.from_numpy(p_ref.astype(np.float32)))
    p_ref = model.flat.cpu().numpy().astype(np.float64)          # start from the fp32 values
    opt = Adam(model, 1e-3)
    for t in range(1, 6):
        g = rng.standard_normal(n) * (0.01 * t)
        model.grad_flat.copy_(torch.from_numpy(g.astype(np.float32)))
        opt.step()
        O.adam_step(p_ref, g.astype(np.float32).astype(np.float64), m_ref, v_ref, t, 1e-3)
    got = model.flat.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(got, p_ref, rtol=0, atol=2e-6)
