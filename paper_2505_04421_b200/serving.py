"""Two-stage serving on B200: per-user KV cache, then cheap candidate scoring.

Mirrors ``longrec.serving`` (pkg/src/longrec/serving.py:84-230): ``build_cache`` /
``score_with_cache`` / ``score_request`` with the same arguments, return values and errors
(``StaleCacheError`` when the model's parameters changed since the build or a candidate's
timestamp differs from the cache's scoring time; ``ConfigError`` for unknown users, mixed
timestamps or a scoring time before the last event).  Beyond the reference's one-user /
one-candidate calls, ``build_caches`` caches many users in one library call and
``score_candidates`` scores ``[users, candidates]`` in one call — the way a server batches.

The cache lives in one device buffer (layout in ``csrc/longer.cu``: cross-layer and per-self-layer
key/value rows in bf16, the last layer's CLS row, the user-side head features, the pad-group
count).  Both stages run in ``_longer_sm100.so``; there is no CPU path.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .errors import ConfigError, EmbeddingLookupError, StaleCacheError
from .inputs import Batch, Candidate, Sample, UserFeatures, tensorize


def _torch():
    import torch
    return torch


@dataclass
class KVCache:
    """Device-resident cache of ``users`` users (serving.py:44-57).  Immutable after build."""

    user_ids: List[int]
    scoring_times: List[int]
    fingerprint: str
    buffer: object               # torch uint8 device tensor of ``nbytes``
    nbytes: int

    @property
    def users(self) -> int:
        return len(self.user_ids)

    # single-user view, as in the reference
    @property
    def user_id(self) -> int:
        return self.user_ids[0]

    @property
    def scoring_time(self) -> int:
        return self.scoring_times[0]


def cache_size_bytes(model, users: int = 1) -> int:
    """Device bytes of a cache of ``users`` users (``longer_cache_bytes``)."""
    n = ctypes.c_size_t()
    _lib.check(model._lib.longer_cache_bytes(ctypes.byref(_lib.dims_of(model.cfg, users)), ctypes.byref(n)))
    return int(n.value)


def build_caches(model, users: Sequence[tuple]) -> KVCache:
    """Stage 1 for many users in one call: ``users`` = [(events, UserFeatures, scoring_time)]."""
    if not users:
        raise ConfigError("build_caches needs at least one user")
    samples = []
    for events, feats, scoring_time in users:
        feats = UserFeatures(feats.uid, feats.profile_bucket)
        samples.append(Sample(tuple(events), feats, Candidate(0, int(scoring_time)), 0))
    host = tensorize(samples, model.cfg)            # range checks + future-event check
    return build_caches_batch(model, host, [int(s.candidate.timestamp) for s in samples])


def build_caches_batch(model, batch: Batch, scoring_times: Sequence[int]) -> KVCache:
    """Stage 1 from an already tensorised batch of users (``dt`` measured from each user's
    scoring time; ``cand_item`` / ``label`` are ignored)."""
    torch = _torch()
    b = model.to_device_batch(batch)
    U = b.size
    if len(scoring_times) != U:
        raise ConfigError("one scoring time per user")
    nbytes = cache_size_bytes(model, U)
    buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=model.device)
    base = (buf.data_ptr() + 255) & ~255
    ws, ws_bytes = model._workspace(U)
    # the cache build runs a forward in the training workspace of batch size U: any pending
    # LongerFunction.backward of that workspace must see its activations as gone
    model._fwd_gen = getattr(model, "_fwd_gen", 0) + 1
    _lib.check(model._lib.longer_cache_build(
        ctypes.byref(_lib.dims_of(model.cfg, U)), ctypes.c_void_p(model.flat.data_ptr()),
        ctypes.byref(model._struct(b)), ctypes.c_void_p(ws), ws_bytes, ctypes.c_void_p(base), nbytes,
        model._stream()))
    model.read_status(U)
    uids = [int(x) for x in (b.uid.cpu().tolist() if hasattr(b.uid, "cpu") else b.uid)]
    cache = KVCache(uids, [int(t) for t in scoring_times], model.fingerprint(), buf, nbytes)
    cache._base = base
    cache._keep = b                                   # inputs stay alive until the stream consumes them
    return cache


def build_cache(model, user_events, user_features: UserFeatures, scoring_time: int) -> KVCache:
    """``build_cache`` (serving.py:84-144): one user's candidate-independent state."""
    return build_caches(model, [(user_events, user_features, scoring_time)])


def _check_fresh(model, cache: KVCache) -> None:
    if cache.fingerprint != model.fingerprint():
        raise StaleCacheError(f"cache fingerprint {cache.fingerprint} != model {model.fingerprint()}; "
                              "rebuild after parameter updates")


def score_candidates(model, cache: KVCache, candidates, check: bool = True) -> "object":
    """Stage 2, batched: ``candidates`` is a [users][C] nested list of ``Candidate`` (every user the
    same C), an int array of item ids [users, C] (then the timestamps are the caches' own), or an
    int tensor of item ids (device or pinned host memory: copied asynchronously, checked on the device).
    Returns probabilities as a device tensor [users, C].  With ``check`` the device-side id check
    is read back (one host sync), as the reference raises ``EmbeddingLookupError`` eagerly."""
    torch = _torch()
    _check_fresh(model, cache)
    U = cache.users
    if torch.is_tensor(candidates):
        # an int tensor of item ids [users, C], on the device or in (pinned) host memory: no host
        # conversion, an asynchronous copy; out-of-range ids are caught by the device-side check
        if candidates.dim() != 2 or candidates.shape[0] != U:
            raise ConfigError(f"candidate ids must be [users={U}, C]")
        if candidates.dtype.is_floating_point or candidates.dtype == torch.bool:
            raise ConfigError("candidate ids must be integers")
        C = int(candidates.shape[1])
        if C == 0:
            return torch.zeros((U, 0), dtype=torch.float32, device=model.device)
        cand_dev = candidates.to(device=model.device, dtype=torch.int32, non_blocking=True).contiguous()
        probs = torch.empty((U, C), dtype=torch.float32, device=model.device)
        base = score_device(model, cache, cand_dev, probs)
        if check:
            flags = ctypes.c_int32()
            _lib.check(model._lib.longer_read_status(ctypes.c_void_p(base), ctypes.byref(flags), model._stream()))
            if flags.value & 1:
                raise EmbeddingLookupError("candidate item id outside the item table")
        return probs
    if isinstance(candidates, np.ndarray) or hasattr(candidates, "dtype"):
        items = np.asarray(candidates.cpu() if hasattr(candidates, "cpu") else candidates, dtype=np.int64)
        if items.ndim != 2 or items.shape[0] != U:
            raise ConfigError(f"candidate ids must be [users={U}, C]")
    else:
        rows = list(candidates)
        if len(rows) != U:
            raise ConfigError(f"expected candidates for {U} users, got {len(rows)}")
        C = len(rows[0]) if rows else 0
        items = np.zeros((U, C), np.int64)
        for u, row in enumerate(rows):
            if len(row) != C:
                raise ConfigError("every user needs the same number of candidates in one call")
            for j, cand in enumerate(row):
                if int(cand.timestamp) != cache.scoring_times[u]:
                    raise StaleCacheError(f"candidate timestamp {cand.timestamp} != cache scoring time "
                                          f"{cache.scoring_times[u]}")
                items[u, j] = cand.item_id
    C = items.shape[1]
    if C == 0:
        return torch.zeros((U, 0), dtype=torch.float32, device=model.device)
    if items.size and (items.min() < 0 or items.max() >= model.cfg.vocab):
        raise EmbeddingLookupError(f"item id out of range [0, {model.cfg.vocab})")
    cand_dev = torch.from_numpy(items.astype(np.int32)).to(model.device, non_blocking=True)
    probs = torch.empty((U, C), dtype=torch.float32, device=model.device)
    base = score_device(model, cache, cand_dev, probs)
    if not check:
        return probs
    flags = ctypes.c_int32()
    _lib.check(model._lib.longer_read_status(ctypes.c_void_p(base), ctypes.byref(flags), model._stream()))
    if flags.value & 1:
        raise EmbeddingLookupError("candidate item id outside the item table")
    return probs


def score_device(model, cache: KVCache, cand_dev, probs) -> int:
    """Stage 2 on device-resident inputs, no host work or sync (graph-capturable): ``cand_dev``
    int32 [users, C] item ids (checked on device: the status flag), ``probs`` float32 [users, C]
    output.  Returns the workspace base address (its first word is the status flag)."""
    torch = _torch()
    U, C = int(cand_dev.shape[0]), int(cand_dev.shape[1])
    if U != cache.users:
        raise ConfigError(f"candidate ids must be [users={cache.users}, C]")
    dims = _lib.dims_of(model.cfg, U)
    key = ("score", U, C)
    if key not in model._ws:
        n = ctypes.c_size_t()
        _lib.check(model._lib.longer_score_workspace_bytes(ctypes.byref(dims), C, ctypes.byref(n)))
        model._ws[key] = torch.zeros(n.value + 256, dtype=torch.uint8, device=model.device)
    ws = model._ws[key]
    base = (ws.data_ptr() + 255) & ~255
    _lib.check(model._lib.longer_cache_score(
        ctypes.byref(dims), ctypes.c_void_p(model.flat.data_ptr()), ctypes.c_void_p(cache._base), cache.nbytes,
        ctypes.c_void_p(cand_dev.data_ptr()), C, ctypes.c_void_p(base), ws.numel() - (base - ws.data_ptr()),
        ctypes.c_void_p(probs.data_ptr()), model._stream()))
    return base


def full_batch_for(users: Batch, cand_items, user: int = 0) -> Batch:
    """The full-forward batch of one cached user paired with each candidate item (checking aid)."""
    n = int(cand_items.shape[0])
    rep = lambda a: a[user:user + 1].repeat_interleave(n, dim=0) if hasattr(a, "repeat_interleave") \
        else np.repeat(np.asarray(a)[user:user + 1], n, axis=0)
    out = {f: rep(getattr(users, f)) for f in Batch.FIELDS}
    out["cand_item"] = cand_items.to(out["items"].device).int() if hasattr(cand_items, "to") else cand_items
    return Batch(**out)


def score_with_cache(model, cache: KVCache, candidate: Candidate) -> float:
    """``score_with_cache`` (serving.py:147-167): one candidate of a one-user cache."""
    _check_fresh(model, cache)
    if cache.users != 1:
        raise ConfigError("score_with_cache takes a single-user cache; use score_candidates")
    if int(candidate.timestamp) != cache.scoring_time:
        raise StaleCacheError(f"candidate timestamp {candidate.timestamp} != cache scoring time "
                              f"{cache.scoring_time}")
    return float(score_candidates(model, cache, [[candidate]])[0, 0].item())


# ----------------------------------------------------------------- request API (serving.py:172-230)
@dataclass
class ScoreRequest:
    user_id: int
    candidates: list             # of Candidate; all share one timestamp


@dataclass
class ScoreResponse:
    user_id: int
    probabilities: list
    cache_build_ns: int
    per_candidate_ns: list

    def to_json_dict(self) -> dict:
        return {"user_id": self.user_id, "probabilities": self.probabilities,
                "cache_build_ns": self.cache_build_ns, "per_candidate_ns": self.per_candidate_ns}


def score_request(model, sample_store: dict, request: ScoreRequest) -> ScoreResponse:
    """Serve one request with a per-user cache; response order = request order
    (serving.py:199-230).  All candidates are scored in ONE device call; ``per_candidate_ns`` is
    that call's time split evenly."""
    if request.user_id not in sample_store:
        raise ConfigError(f"unknown user_id {request.user_id}")
    base = sample_store[request.user_id]
    if request.candidates:
        stamps = {c.timestamp for c in request.candidates}
        if len(stamps) > 1:
            raise ConfigError("candidates in one request must share a timestamp")
        scoring_time = request.candidates[0].timestamp
    else:
        scoring_time = base.candidate.timestamp
    if base.events and base.events[-1].timestamp > scoring_time:
        raise ConfigError("scoring time precedes the last user event")
    torch = _torch()
    t0 = time.perf_counter_ns()
    cache = build_cache(model, base.events, base.user_features, scoring_time)
    torch.cuda.synchronize(model.device)
    build_ns = time.perf_counter_ns() - t0
    probs, times = [], []
    if request.candidates:
        t1 = time.perf_counter_ns()
        p = score_candidates(model, cache, [list(request.candidates)])
        probs = [float(x) for x in p[0].cpu().tolist()]
        dt = time.perf_counter_ns() - t1
        times = [dt // len(probs)] * len(probs)
    return ScoreResponse(request.user_id, probs, build_ns, times)
