"""Two-stage serving (KV cache) on the sm_100a path, through the C ABI.

* golden vectors from the reference's own ``build_cache`` / ``score_with_cache``
  (tests/golden/serving_*.npz, pkg/src/longrec/serving.py:84-167);
* cached scores ≡ this library's full forward of the same (user, candidate) samples — the
  reference asserts this identity at 1e-9 in float64; here both sides are bf16-operand paths that
  differ only in summation order (own key last, separate GEMM row sets), tolerance 2e-3;
* the float64 oracle at the c2 shape (L=2000, d=32, InnerTrans) with mixed history lengths;
* the reference's errors: StaleCacheError (parameters changed, candidate timestamp ≠ scoring
  time), EmbeddingLookupError (candidate id), ConfigError (request validation).
Tolerance vs reference/oracle as for the forward: |Δp| ≤ 5e-3.
"""
import glob
import json
import os

import numpy as np
import pytest

from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig, StaleCacheError, EmbeddingLookupError, ConfigError
from paper_2505_04421_b200.inputs import Batch, Candidate, Sample, UserFeatures, synthetic_samples, tensorize

pytestmark = pytest.mark.gpu

SERVING = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "serving_*.npz")))


def _model(cfg, P, seed=0):
    from paper_2505_04421_b200.model import LongerModel
    m = LongerModel(cfg, seed=seed)
    if P is not None:
        m.load_params(P)
    return m


def _expand(users: Batch, cand: np.ndarray) -> Batch:
    """Full-forward batch of every (user, candidate) pair, user-major."""
    U, C = cand.shape
    rep = lambda a: np.repeat(np.asarray(a), C, axis=0)
    return Batch(rep(users.items), rep(users.actions), rep(users.dt), rep(users.n_events), rep(users.uid),
                 rep(users.profile), cand.reshape(-1).astype(np.int32), np.zeros(U * C, np.float32))


@pytest.mark.parametrize("path", SERVING, ids=[os.path.basename(p)[:-4] for p in SERVING])
def test_cached_scores_match_reference_golden(path):
    from paper_2505_04421_b200 import serving as S
    z = np.load(path)
    cfg = ModelConfig(**json.loads(str(z["cfg"])))
    P = {k[2:]: z[k] for k in z.files if k.startswith("P/")}
    users = Batch(**{k[6:]: z[k] for k in z.files if k.startswith("users/")})
    cand = z["cand"]
    model = _model(cfg, P)
    cache = S.build_caches_batch(model, users, [int(t) for t in z["scoring_time"]])
    p = S.score_candidates(model, cache, cand).cpu().numpy().astype(np.float64)
    assert p.shape == cand.shape
    assert np.max(np.abs(p - z["p_cached"])) <= 5e-3, np.abs(p - z["p_cached"])
    # ≡ this library's own full forward of the expanded (user, candidate) batch
    pf = model.forward(_expand(users, cand)).cpu().numpy().reshape(cand.shape)
    assert np.max(np.abs(p - pf)) <= 2e-3, np.abs(p - pf)


C2 = dict(L=2000, d=32, K=4, k=32, N=2, m=3, merge_mode="inner")


@pytest.mark.parametrize("kw,n_events", [
    (C2, [2000, 700, 5]),
    (dict(C2, merge_mode="concat", heads=2), [2000, 31]),
    # c5 widths (D = 256, K = 8): the cached attention at head width 256 on the SIMT kernel
    (dict(L=96, d=32, K=8, k=4, N=2, m=3, merge_mode="inner"), [96, 40]),
])
def test_cached_scores_match_oracle_c2(kw, n_events):
    from paper_2505_04421_b200 import serving as S
    from paper_2505_04421_b200.params import init_params
    cfg = ModelConfig(**kw).validate()
    rng = np.random.default_rng(5)
    P = {n: a + 0.02 * rng.standard_normal(a.shape) for n, a in init_params(cfg, seed=0).items()}
    base = []
    for i, n in enumerate(n_events):
        s = synthetic_samples(cfg, 1, seed=40 + i, n_events=n)[0]
        base.append(s)
    C = 3
    cand = rng.integers(cfg.vocab, size=(len(base), C)).astype(np.int32)
    model = _model(cfg, P)
    cache = S.build_caches(model, [(s.events, s.user_features, s.candidate.timestamp) for s in base])
    p = S.score_candidates(model, cache, [[Candidate(int(c), s.candidate.timestamp) for c in row]
                                          for s, row in zip(base, cand)]).cpu().numpy()
    samples = [Sample(s.events, s.user_features, Candidate(int(c), s.candidate.timestamp), 0)
               for s, row in zip(base, cand) for c in row]
    p_ref, _ = O.forward(P, cfg, tensorize(samples, cfg).as_dict())
    assert np.max(np.abs(p.reshape(-1) - p_ref)) <= 5e-3, np.abs(p.reshape(-1) - p_ref)


def test_many_users_many_candidates_equal_full_forward():
    """A server-sized call (64 users × 96 candidates, c1 widths) against the full forward."""
    from paper_2505_04421_b200 import serving as S
    cfg = ModelConfig(L=256, d=16, K=4, k=16, N=1, m=3).validate()
    model = _model(cfg, None, seed=3)
    samples = synthetic_samples(cfg, 64, seed=9)
    users = tensorize([Sample(s.events, s.user_features, Candidate(0, s.candidate.timestamp), 0)
                       for s in samples], cfg)
    cand = np.random.default_rng(1).integers(cfg.vocab, size=(64, 96)).astype(np.int32)
    cache = S.build_caches_batch(model, users, [s.candidate.timestamp for s in samples])
    p = S.score_candidates(model, cache, cand).cpu().numpy()
    pf = model.forward(_expand(users, cand)).cpu().numpy().reshape(cand.shape)
    assert np.max(np.abs(p - pf)) <= 2e-3


@pytest.mark.parametrize("heads,qk_gain", [(1, 1.0), (1, 6.0), (4, 6.0)], ids=["dh128", "dh128-sharp", "dh32-sharp"])
def test_c2_partial_tiles_and_rescaled_softmax_equal_full_forward(heads, qk_gain):
    """c2 widths (502 cached cross keys = 4 key chunks of 128), 3 users × 300 candidates (a partial
    128-candidate tile and a partial 8-row head group), mixed history lengths.  qk_gain scales the
    query / key projections so that the scores spread over tens of units: the single-pass cached
    attention must then move its running max (and rescale O in TMEM) between key chunks."""
    from paper_2505_04421_b200 import serving as S
    from paper_2505_04421_b200.params import init_params
    cfg = ModelConfig(**dict(C2, heads=heads)).validate()
    P = init_params(cfg, seed=0)
    rng = np.random.default_rng(7)
    for name in list(P):
        if name.endswith(("w_q", "w_k")):
            P[name] = P[name] * qk_gain
        elif name.startswith("tables."):
            P[name] = P[name] + 0.05 * rng.standard_normal(P[name].shape)
    model = _model(cfg, P)
    samples = [synthetic_samples(cfg, 1, seed=70 + i, n_events=n)[0] for i, n in enumerate([2000, 900, 17])]
    users = tensorize([Sample(s.events, s.user_features, Candidate(0, s.candidate.timestamp), 0)
                       for s in samples], cfg)
    cand = rng.integers(cfg.vocab, size=(3, 300)).astype(np.int32)
    cache = S.build_caches_batch(model, users, [s.candidate.timestamp for s in samples])
    p = S.score_candidates(model, cache, cand).cpu().numpy()
    pf = model.forward(_expand(users, cand)).cpu().numpy().reshape(cand.shape)
    assert np.max(np.abs(p - pf)) <= 3e-3, np.abs(p - pf).max()


def test_single_user_api_and_errors():
    from paper_2505_04421_b200 import serving as S
    cfg = ModelConfig(L=64, d=16, K=4, k=8, N=2, m=3, merge_mode="inner", n_users=64).validate()
    model = _model(cfg, None, seed=1)
    s = synthetic_samples(cfg, 1, seed=2)[0]
    cache = S.build_cache(model, s.events, s.user_features, s.candidate.timestamp)
    p = S.score_with_cache(model, cache, s.candidate)
    full = model.score(s)
    assert abs(p - full) <= 2e-3
    with pytest.raises(StaleCacheError):
        S.score_with_cache(model, cache, Candidate(s.candidate.item_id, s.candidate.timestamp + 1))
    with pytest.raises(EmbeddingLookupError):
        S.score_with_cache(model, cache, Candidate(cfg.vocab, s.candidate.timestamp))
    with pytest.raises(ConfigError):      # future event relative to the scoring time
        S.build_cache(model, s.events, s.user_features, s.events[-1].timestamp - 1)
    # parameters change → the cache is stale
    model.load_params({"head.b2": np.array([0.5], np.float32)})
    with pytest.raises(StaleCacheError):
        S.score_with_cache(model, cache, s.candidate)


def test_score_request():
    from paper_2505_04421_b200 import serving as S
    cfg = ModelConfig(L=64, d=16, K=4, k=8, N=1, m=3, n_users=64).validate()
    model = _model(cfg, None, seed=4)
    store = {i: s for i, s in enumerate(synthetic_samples(cfg, 3, seed=6))}
    ts = store[1].candidate.timestamp
    cands = [Candidate(i, ts) for i in (5, 17, 3, 99)]
    resp = S.score_request(model, store, S.ScoreRequest(1, cands))
    assert resp.user_id == 1 and len(resp.probabilities) == 4 and len(resp.per_candidate_ns) == 4
    for c, p in zip(cands, resp.probabilities):
        full = model.score(Sample(store[1].events, store[1].user_features, c, 0))
        assert abs(p - full) <= 2e-3
    assert set(resp.to_json_dict()) == {"user_id", "probabilities", "cache_build_ns", "per_candidate_ns"}
    with pytest.raises(ConfigError):
        S.score_request(model, store, S.ScoreRequest(7, cands))
    with pytest.raises(ConfigError):
        S.score_request(model, store, S.ScoreRequest(1, [Candidate(1, ts), Candidate(2, ts + 1)]))
    empty = S.score_request(model, store, S.ScoreRequest(2, []))
    assert empty.probabilities == []


@pytest.mark.parametrize("strategy", ["uniform", "recent_uniform", "learnable"])
def test_cached_scores_other_query_strategies(strategy):
    """Cached scoring ≡ the full forward for the non-"recent" query sets."""
    from paper_2505_04421_b200 import serving as S
    cfg = ModelConfig(L=256, d=16, K=4, k=16, N=2, m=3, query_strategy=strategy).validate()
    model = _model(cfg, None, seed=7)
    samples = synthetic_samples(cfg, 6, seed=12)
    samples = [Sample(s.events[:n], s.user_features, Candidate(0, s.candidate.timestamp), 0)
               for s, n in zip(samples, [256, 200, 90, 40, 9, 0])]
    users = tensorize(samples, cfg)
    cand = np.random.default_rng(2).integers(cfg.vocab, size=(6, 8)).astype(np.int32)
    cache = S.build_caches_batch(model, users, [s.candidate.timestamp for s in samples])
    p = S.score_candidates(model, cache, cand).cpu().numpy()
    pf = model.forward(_expand(users, cand)).cpu().numpy().reshape(cand.shape)
    assert np.max(np.abs(p - pf)) <= 2e-3, np.abs(p - pf)


def test_tensor_candidate_ids():
    """Candidate ids as a torch tensor (pinned host or device memory: asynchronous copy, no host
    conversion) score like the numpy array, and an out-of-range id raises through the device flag."""
    import torch
    from paper_2505_04421_b200 import serving as S
    cfg = ModelConfig(L=64, d=16, K=4, k=8, N=2, m=3, merge_mode="inner", n_users=64).validate()
    model = _model(cfg, None, seed=1)
    base = synthetic_samples(cfg, 3, seed=9)
    cache = S.build_caches(model, [(s.events, s.user_features, s.candidate.timestamp) for s in base])
    ids = np.random.default_rng(2).integers(0, cfg.vocab, size=(3, 5)).astype(np.int32)
    p_np = S.score_candidates(model, cache, ids).cpu().numpy()
    p_host = S.score_candidates(model, cache, torch.from_numpy(ids).pin_memory()).cpu().numpy()
    p_dev = S.score_candidates(model, cache, torch.from_numpy(ids).to("cuda").long()).cpu().numpy()
    np.testing.assert_array_equal(p_host, p_np)
    np.testing.assert_array_equal(p_dev, p_np)
    bad = ids.copy()
    bad[1, 2] = cfg.vocab
    with pytest.raises(EmbeddingLookupError):
        S.score_candidates(model, cache, torch.from_numpy(bad).to("cuda"))
    with pytest.raises(ConfigError):
        S.score_candidates(model, cache, torch.zeros((2, 5), dtype=torch.int32))
