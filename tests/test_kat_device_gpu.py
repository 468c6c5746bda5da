"""Integer, error and invariance known-answer tests of the reference suite, run on the device path.

* time buckets (pkg/tests/test_inputs.py:93-106, pkg/src/longrec/inputs.py:307-315): the bucket the
  device computes, observed bit-exactly two ways — (1) in the backward, the only rows of
  time_bucket_table's gradient that are not exactly 0 are the events' bucket and 0 (the target
  token's zero delta, inputs.py:500-512); (2) in the forward, the token-MLP output h depends on
  the delta only through the bucket (bit-identical within a bucket, different across buckets).
  Fused and per-stage front-end, n_time_buckets 32 and 8, deltas up to 2^40 (host-clamped to
  int32, exact because buckets clamp at <= 31);
* EmbeddingLookupError from the device flag (inputs.py:406-411) for every id kind, never clamped
  silently; ConfigError for a negative delta; both also through the deferred (async) check;
* NumericalError for a non-finite loss (pkg/src/longrec/model.py:563-566);
* LayerNorm of a constant row is exactly its bias (pkg/tests/test_tensors.py:159-161);
* target-row and causal-prefix invariance, bit-exact, of every activation of the trace
  (pkg/tests/test_attention.py:216-250, pkg/tests/test_model.py:100-109).
"""
import ctypes

import numpy as np
import pytest

from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, synthetic_batch
from paper_2505_04421_b200.errors import ConfigError, EmbeddingLookupError, NumericalError
from paper_2505_04421_b200.inputs import Batch, Candidate, Event, Sample, UserFeatures, tensorize

pytestmark = pytest.mark.gpu

SMALL = dict(L=64, d=16, K=4, k=4, N=1, m=3, merge_mode="inner", n_users=50, vocab=60)
# reference KATs (test_inputs.py:93-106) + the power-of-two boundaries up to the int32 range
REF_KAT = {3601: 12, 0: 0, 1: 1, 2: 2, 2 ** 40: 31}
DELTAS = sorted(set(list(REF_KAT) + [2 ** (b - 1) for b in range(1, 32)] + [2 ** b - 1 for b in range(1, 32)]
                    + [3, 5, 900, 86_400, 2 ** 31 - 1, 2 ** 35]))


def _model(cfg, P=None):
    from paper_2505_04421_b200.model import LongerModel
    m = LongerModel(cfg, seed=0)
    if P is not None:
        m.load_params(P)
    return m


def _samples_with_delta(cfg, delta, n=3, seed=0):
    """n samples whose every event lies exactly `delta` seconds before the candidate."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        cand_ts = 2 ** 41 + 10_000
        ne = cfg.L - 5 * i
        ev = tuple(Event(int(rng.integers(cfg.vocab)), int(rng.integers(cfg.n_actions)), cand_ts - delta)
                   for _ in range(ne))
        out.append(Sample(ev, UserFeatures(int(rng.integers(cfg.n_users)), int(rng.integers(cfg.n_profiles))),
                          Candidate(int(rng.integers(cfg.vocab)), cand_ts), i % 2))
    return out


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("nb", [32, 8])
def test_time_buckets_on_device(fused, nb, monkeypatch):
    monkeypatch.setenv("LONGER_FUSED", fused)
    cfg = ModelConfig(**dict(SMALL, n_time_buckets=nb)).validate()
    model = _model(cfg)
    for dt, want in REF_KAT.items():                         # the oracle restates the reference KATs
        assert int(O.time_bucket(np.array([dt]), 32)[0]) == want
    h_by_bucket = {}
    for delta in DELTAS:
        want = int(O.time_bucket(np.array([delta]), nb)[0])
        if delta in REF_KAT and nb == 32:
            assert want == REF_KAT[delta]
        batch = tensorize(_samples_with_delta(cfg, delta), cfg)
        # (1) backward: exact zero rows everywhere but {bucket, 0}
        model.loss_backward(batch)
        g_time = dict(model.grads())["tables.time_bucket_table"].cpu().numpy()
        nz = set(np.flatnonzero(np.any(g_time != 0.0, axis=1)).tolist())
        assert nz == {want, 0}, (delta, want, nz)
        # (2) forward: h depends on the delta only through its bucket
        _, traces = model.forward_traces(batch)
        h = np.stack([t.h for t in traces])
        if want in h_by_bucket:
            np.testing.assert_array_equal(h, h_by_bucket[want], err_msg=f"delta {delta}")
        else:
            for other in h_by_bucket.values():
                assert np.any(h != other), f"delta {delta}: bucket {want} looks like another bucket"
            h_by_bucket[want] = h
    assert set(h_by_bucket) == set(range(min(nb, 32)))


def _device_batch(cfg, B=4, **bad):
    b = synthetic_batch(cfg, B, seed=3)
    d = {f: np.array(getattr(b, f), copy=True) for f in Batch.FIELDS}
    for f, (idx, val) in bad.items():
        d[f][idx] = val
    return Batch(**d).to("cuda")       # device batch: skips the host-side check entirely


@pytest.mark.parametrize("field,idx,val,exc", [
    ("items", (1, -1), 60, EmbeddingLookupError),      # item id == vocab
    ("items", (2, -3), -1, EmbeddingLookupError),
    ("actions", (0, -2), 4, EmbeddingLookupError),
    ("uid", 3, 50, EmbeddingLookupError),
    ("profile", 0, 16, EmbeddingLookupError),
    ("cand_item", 1, 99, EmbeddingLookupError),
    ("dt", (0, -1), -5, ConfigError),                  # future event
])
@pytest.mark.parametrize("fused", ["1", "0"])
def test_device_flag_raises_reference_errors(field, idx, val, exc, fused, monkeypatch):
    monkeypatch.setenv("LONGER_FUSED", fused)
    cfg = ModelConfig(**SMALL).validate()
    model = _model(cfg)
    good = _device_batch(cfg)
    bad = _device_batch(cfg, **{field: (idx, val)})
    model.loss_backward(good)                          # clean
    with pytest.raises(exc):
        model.loss_backward(bad)
    model.loss_backward(good)                          # flags were reset
    with pytest.raises(exc):
        model.forward(bad, sync_check=True)
    # deferred check: raised by this or a later call, once the step's flags reach the host
    with pytest.raises(exc):
        model.loss_backward(bad, check="async")
        for _ in range(3):
            model.loss_backward(good, check="async")
        model.poll_checks(block=True)
    model.poll_checks(block=True)                      # drained: nothing left to raise


def test_host_check_raises_before_launch():
    cfg = ModelConfig(**SMALL).validate()
    s = _samples_with_delta(cfg, 100, n=1)[0]
    bad = Sample(s.events[:-1] + (Event(cfg.vocab, 0, s.events[-1].timestamp),), s.user_features, s.candidate, 0)
    with pytest.raises(EmbeddingLookupError):
        tensorize([bad], cfg)
    fut = Sample(s.events, s.user_features, Candidate(s.candidate.item_id, s.events[-1].timestamp - 1), 0)
    with pytest.raises(ConfigError):
        tensorize([fut], cfg)


@pytest.mark.parametrize("check", [True, "async"])
def test_non_finite_loss_raises_numerical_error(check):
    cfg = ModelConfig(**SMALL).validate()
    from paper_2505_04421_b200.params import init_params
    P = init_params(cfg, seed=0)
    P["head.b2"] = P["head.b2"] + np.nan
    model = _model(cfg, P)
    batch = synthetic_batch(cfg, 4, seed=1)
    with pytest.raises(NumericalError):
        model.loss_backward(batch, check=check)
        model.poll_checks(block=True)


@pytest.mark.parametrize("W", [16, 32, 128, 256])
def test_layernorm_constant_row_is_its_bias(W):
    """LN(x)·g + b of a constant row is exactly b (the reference KAT with b = 0 gives exact zeros).
    The constants are dyadic: the fp32 row mean is then exact (the reference's 3.3 over 4 float64
    columns happens to be exact too; 32 fp32 copies of 3.3 do not sum exactly)."""
    import torch
    from paper_2505_04421_b200 import _lib
    lib = _lib.load()
    rows = 64
    vals = torch.tensor([3.25, -0.75, 0.0, 1024.0, 2.0 ** -13], dtype=torch.float64)
    x = vals.repeat_interleave(rows // len(vals) + 1)[:rows, None].expand(rows, W).contiguous().float().cuda()
    g = torch.randn(W, device="cuda")
    for b in (torch.zeros(W, device="cuda"), torch.randn(W, device="cuda")):
        y = torch.empty(rows, W, dtype=torch.bfloat16, device="cuda")
        mean = torch.empty(rows, device="cuda")
        rstd = torch.empty(rows, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        assert lib.longer_test_layernorm(ctypes.c_void_p(x.data_ptr()), rows, W, ctypes.c_void_p(g.data_ptr()),
                                         ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                         ctypes.c_void_p(mean.data_ptr()), ctypes.c_void_p(rstd.data_ptr()),
                                         ctypes.c_void_p(st)) == 0
        torch.cuda.synchronize()
        want = b.to(torch.bfloat16).expand(rows, W)
        assert torch.equal(y, want), (y - want.float()).abs().max()


C2_SMALL = dict(L=512, d=32, K=4, k=32, N=2, m=3)


@pytest.mark.parametrize("merge", ["inner", "concat"])
@pytest.mark.parametrize("qs", ["recent", "uniform"])
def test_target_row_invariance(merge, qs):
    """Changing the candidate changes only the target row of every layer; h, merged and every
    other row of every block output are bit-identical (model.py:100-109 / attention.py:216-233)."""
    cfg = ModelConfig(**dict(C2_SMALL, merge_mode=merge, query_strategy=qs)).validate()
    model = _model(cfg)
    b = synthetic_batch(cfg, 5, seed=8, min_events=40)
    other = Batch(**{f: np.array(getattr(b, f), copy=True) for f in Batch.FIELDS})
    other.cand_item = ((other.cand_item + 7) % cfg.vocab).astype(np.int32)
    _, ta = model.forward_traces(b)
    _, tb = model.forward_traces(other)
    for x, y in zip(ta, tb):
        for u, v in zip(x.sequence_branch(), y.sequence_branch()):
            np.testing.assert_array_equal(u, v)
        assert all(np.any(u[-1] != v[-1]) for u, v in zip(x.layers, y.layers))


@pytest.mark.parametrize("merge", ["inner", "concat"])
def test_causal_prefix_invariance(merge):
    """Rewriting the newest event changes merged group G-1 only; every sequence query of an older
    group is bit-identical in every layer (attention.py:236-250) and the newest query changes.
    (The globals see the whole sequence too, but one changed key among ~500 can vanish in the
    bf16 rounding of their attention output, so they are not asserted to change.)"""
    cfg = ModelConfig(**dict(C2_SMALL, merge_mode=merge)).validate()
    model = _model(cfg)
    b = synthetic_batch(cfg, 4, seed=12, min_events=200)
    other = Batch(**{f: np.array(getattr(b, f), copy=True) for f in Batch.FIELDS})
    other.items[:, -1] = (other.items[:, -1] + 1) % cfg.vocab
    _, ta = model.forward_traces(b)
    _, tb = model.forward_traces(other)
    k = cfg.k
    for x, y in zip(ta, tb):
        np.testing.assert_array_equal(x.h[:-1], y.h[:-1])
        assert np.any(x.h[-1] != y.h[-1])
        np.testing.assert_array_equal(x.merged[:-1], y.merged[:-1])
        for u, v in zip(x.layers, y.layers):
            np.testing.assert_array_equal(u[:k - 1], v[:k - 1])
            assert np.any(u[k - 1] != v[k - 1])


def test_trace_matches_oracle():
    """forward(sample) → (p, ForwardTrace) like LongRecModel.forward (model.py:365-372): every
    traced stage against the oracle's intermediate activations."""
    cfg = ModelConfig(**dict(C2_SMALL, merge_mode="inner", query_strategy="uniform")).validate()
    from paper_2505_04421_b200.params import init_params
    P = init_params(cfg, seed=0)
    model = _model(cfg, P)
    b = synthetic_batch(cfg, 3, seed=2, min_events=50)
    p_ref, cache = O.forward(P, cfg, b.as_dict())
    p, traces = model.forward_traces(b)
    np.testing.assert_allclose(p, p_ref, atol=5e-3)
    npg = (cfg.L_padded - np.asarray(b.n_events)) // cfg.K
    qg = O.query_groups(cfg, npg)
    extra = cfg.L_padded - cfg.L

    def close(got, ref, what):                           # bf16 operands, fp32 accumulation
        err = np.abs(got - ref).max() / (np.abs(ref).max() + 1e-12)
        assert err <= 2e-2, (what, err)

    for i, t in enumerate(traces):
        close(t.h, cache["h"][i, extra:], "h")
        close(t.merged, cache["merged"][i], "merged")
        for j, layer in enumerate(t.layers):
            close(layer, cache["layers"][j][i], f"layer {j}")
        close(t.head_input[0], cache["hin"][i], "head_input")
        np.testing.assert_array_equal(t.query_indices, qg[i])
        np.testing.assert_array_equal(t.query_positions[:cfg.k], qg[i] * cfg.K + cfg.K - 1)
        assert t.h.shape == (cfg.L, cfg.d) and t.merged.shape == (cfg.merged_len, cfg.D)
        assert len(t.layers) == 1 + cfg.N and t.head_input.shape == (1, 4 * cfg.D + 2 * cfg.d)
    # a single Sample goes through the same path
    from paper_2505_04421_b200.inputs import synthetic_samples
    s = synthetic_samples(cfg, 1, seed=4, n_events=77)[0]
    p1, tr = model.forward(s)
    assert isinstance(p1, float) and abs(p1 - tr.p) < 1e-7
    p_ref1, _ = O.forward(P, cfg, tensorize([s], cfg).as_dict())
    assert abs(p1 - float(p_ref1[0])) <= 5e-3
