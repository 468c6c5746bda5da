"""Sample records and their tensorisation into the device batch layout.

``Event``/``UserFeatures``/``Candidate``/``Sample`` mirror the reference records
(``pkg/src/longrec/inputs.py:35-99``) so reference datasets drop in unchanged.

``Batch`` is the layout the C-ABI consumes (``include/longer.h`` ``LongerBatch``): token
arrays ``[B, L]`` right-aligned exactly like ``encode_events`` (``inputs.py:457-482``: keep the
last L events, left-pad), plus per-sample scalars.  Time deltas are ``candidate_ts - event_ts``
in seconds; the device computes the log2 bucket (``inputs.py:307-315``).  Because buckets clamp
at ``n_time_buckets - 1 <= 31``, clamping deltas to int32 max is exact.
"""
from __future__ import annotations

import gzip
import json
import threading
from dataclasses import dataclass
from itertools import chain
from operator import attrgetter
from typing import Optional, Sequence

import numpy as np

from .config import ModelConfig
from .errors import ConfigError, EmbeddingLookupError

INT32_MAX = 2 ** 31 - 1


@dataclass(frozen=True)
class Event:
    item_id: int
    action_type: int
    timestamp: int


@dataclass(frozen=True)
class UserFeatures:
    uid: int
    profile_bucket: int


@dataclass(frozen=True)
class Candidate:
    item_id: int
    timestamp: int


@dataclass(frozen=True)
class Sample:
    """One training record (pkg/src/longrec/inputs.py:55-100): ordered events, user features,
    candidate, label.  Same JSON record layout as the reference."""

    events: tuple
    user_features: UserFeatures
    candidate: Candidate
    label: int

    def validate(self, L_max: Optional[int] = None) -> "Sample":
        ts = [e.timestamp for e in self.events]
        if any(a > b for a, b in zip(ts, ts[1:])):
            raise ConfigError("events must be sorted non-decreasing by timestamp")
        if ts and ts[-1] > self.candidate.timestamp:
            raise ConfigError("event timestamps must not exceed the candidate timestamp")
        if L_max is not None and len(self.events) > L_max:
            raise ConfigError(f"sample has {len(self.events)} events > L_max={L_max}")
        if self.label not in (0, 1):
            raise ConfigError("label must be 0 or 1")
        return self

    def to_json_dict(self) -> dict:
        return {
            "events": [{"item_id": e.item_id, "action_type": e.action_type, "timestamp": e.timestamp}
                       for e in self.events],
            "user_features": {"uid": self.user_features.uid,
                              "profile_bucket": self.user_features.profile_bucket},
            "candidate": {"item_id": self.candidate.item_id, "timestamp": self.candidate.timestamp},
            "label": self.label,
        }

    @classmethod
    def from_json_dict(cls, rec: dict) -> "Sample":
        return cls(events=tuple(Event(e["item_id"], e["action_type"], e["timestamp"]) for e in rec["events"]),
                   user_features=UserFeatures(rec["user_features"]["uid"], rec["user_features"]["profile_bucket"]),
                   candidate=Candidate(rec["candidate"]["item_id"], rec["candidate"]["timestamp"]),
                   label=int(rec["label"]))


@dataclass
class Dataset:
    """Samples of a JSONL file (pkg/src/longrec/inputs.py:103-119)."""

    samples: list

    def __len__(self) -> int:
        return len(self.samples)

    def labels(self) -> np.ndarray:
        return np.array([s.label for s in self.samples], dtype=np.int64)

    def tensorized(self, cfg: ModelConfig) -> Batch:
        """The whole dataset in the C-ABI layout (host numpy, checked once), cached per L."""
        cache = self.__dict__.setdefault("_columns", {})
        if cfg.L not in cache:
            cache[cfg.L] = tensorize(self.samples, cfg)
        return cache[cfg.L]

    def batches(self, cfg: ModelConfig, batch_size: int, pin: bool = True, device=None, prefetch: int = 2,
                shuffle: bool = False, seed: int = 0):
        """``Batch``es of ``batch_size`` samples (file order, or a seeded permutation with
        ``shuffle``), sliced from the tensorised dataset.  ``pin``: host batches in pinned memory.
        ``device``: a background thread slices, pins and copies the next ``prefetch`` batches
        host→device on its own CUDA stream while the caller's step runs; each yielded device batch
        is ready on the caller's current stream (it waits on the copy's event)."""
        cols = self.tensorized(cfg)
        N = len(self)
        order = np.random.default_rng(seed).permutation(N) if shuffle else None

        def host(i):
            idx = slice(i, min(i + batch_size, N)) if order is None else order[i:i + batch_size]
            b = Batch(**{f: np.ascontiguousarray(getattr(cols, f)[idx]) for f in Batch.FIELDS})
            return b.pin() if (pin or device is not None) else b

        starts = range(0, N, batch_size)
        if device is None:
            for i in starts:
                yield host(i)
            return
        yield from _prefetched(host, starts, device, prefetch)


def _prefetched(host, starts, device, depth):
    """Background host slicing + pinned H2D on a side stream, ``depth`` batches ahead."""
    import queue

    import torch
    q = queue.Queue(maxsize=max(1, depth))
    stream = torch.cuda.Stream(device)
    stop = threading.Event()

    def work():
        try:
            for i in starts:
                if stop.is_set():
                    break
                hb = host(i)
                with torch.cuda.stream(stream):
                    db = hb.to(device, non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(stream)
                q.put((db, ev, hb))
        except BaseException as exc:           # surfaced on the consumer side
            q.put(exc)
        q.put(None)

    t = threading.Thread(target=work, daemon=True)
    t.start()
    try:
        while True:
            item = q.get()
            if item is None:
                break
            if isinstance(item, BaseException):
                raise item
            db, ev, hb = item
            torch.cuda.current_stream(device).wait_event(ev)
            yield db
    finally:
        stop.set()


def save_dataset(dataset: Dataset, path: str) -> None:
    """Newline-delimited JSON, one sample per line; ``.gz`` compresses (inputs.py:279-285)."""
    opener = gzip.open if str(path).endswith(".gz") else open
    with opener(path, "wt", encoding="utf-8") as fh:
        for smp in dataset.samples:
            fh.write(json.dumps(smp.to_json_dict(), separators=(",", ":")))
            fh.write("\n")


def load_dataset(path: str, L_max: Optional[int] = None) -> Dataset:
    """Read a reference JSONL dataset (inputs.py:288-301), validating every record."""
    opener = gzip.open if str(path).endswith(".gz") else open
    samples = []
    with opener(path, "rt", encoding="utf-8") as fh:
        for line in fh:
            line = line.strip()
            if not line:
                continue
            try:
                samples.append(Sample.from_json_dict(json.loads(line)).validate(L_max))
            except (KeyError, TypeError, json.JSONDecodeError) as exc:
                raise ConfigError(f"malformed dataset record: {exc}") from exc
    return Dataset(samples)


@dataclass
class Batch:
    """Host (numpy) or device (torch) arrays in the C-ABI batch layout."""

    items: object       # int32 [B, L]
    actions: object     # int32 [B, L]
    dt: object          # int32 [B, L]   candidate_ts - event_ts, clamped to int32
    n_events: object    # int32 [B]      real events (<= L), right-aligned
    uid: object         # int32 [B]
    profile: object     # int32 [B]
    cand_item: object   # int32 [B]
    label: object       # float32 [B]

    FIELDS = ("items", "actions", "dt", "n_events", "uid", "profile", "cand_item", "label")

    @property
    def size(self) -> int:
        return int(self.n_events.shape[0])

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f in self.FIELDS}

    def to(self, device, non_blocking: bool = True) -> "Batch":
        import torch
        out = {}
        for f in self.FIELDS:
            v = getattr(self, f)
            if isinstance(v, np.ndarray):
                v = torch.from_numpy(np.ascontiguousarray(v))
            out[f] = v.to(device, non_blocking=non_blocking)
        return Batch(**out)

    def pin(self) -> "Batch":
        import torch
        out = {}
        for f in self.FIELDS:
            v = getattr(self, f)
            if isinstance(v, np.ndarray):
                v = torch.from_numpy(np.ascontiguousarray(v))
            out[f] = v.pin_memory()
        return Batch(**out)

    def nbytes(self) -> int:
        return int(sum(getattr(self, f).nbytes for f in self.FIELDS))


def _check_ids(name: str, arr: np.ndarray, rows: int) -> None:
    """``_checked_ids`` (pkg/src/longrec/inputs.py:406-411): never clamp."""
    if arr.size and (arr.min() < 0 or arr.max() >= rows):
        raise EmbeddingLookupError(f"{name} id out of range [0, {rows}): {arr.min()}..{arr.max()}")


def tensorize(samples: Sequence[Sample], cfg: ModelConfig, check: bool = True) -> Batch:
    """Samples → ``Batch`` (host numpy).  Raises the reference's errors for bad input.

    The event fields are pulled from all events of the batch by one C-level iterator chain
    (≈ 1.5 M attribute reads for 256 x 2000 events: this, not the placement, bounds it), then placed
    into the right-aligned [B, L] grid and range-checked with vector operations.  Training loops
    should tensorise a dataset once (``Dataset.tensorized``) and slice batches from it
    (``Dataset.batches``)."""
    B, L = len(samples), cfg.L
    evs = [tuple(s.events)[-L:] for s in samples]
    n = np.fromiter((len(e) for e in evs), np.int64, B)
    tot = int(n.sum())
    fields = attrgetter("item_id", "action_type", "timestamp")   # one pass, three reads per event
    flat = np.fromiter(chain.from_iterable(map(fields, chain.from_iterable(evs))), np.int64,
                       3 * tot).reshape(tot, 3)
    cand_ts = np.fromiter((s.candidate.timestamp for s in samples), np.int64, B)
    rows = np.repeat(np.arange(B), n)
    starts = np.cumsum(n) - n
    cols = np.arange(tot) - np.repeat(starts, n) + np.repeat(L - n, n)
    delta = np.repeat(cand_ts, n) - flat[:, 2]
    if check:
        _check_ids("item", flat[:, 0], cfg.vocab)
        _check_ids("action", flat[:, 1], cfg.n_actions)
        if (delta < 0).any():
            raise ConfigError("future event: negative time delta")
    items = np.zeros((B, L), np.int32)
    actions = np.zeros((B, L), np.int32)
    dt = np.zeros((B, L), np.int32)
    items[rows, cols] = flat[:, 0]
    actions[rows, cols] = flat[:, 1]
    dt[rows, cols] = np.minimum(delta, INT32_MAX)
    uid = np.fromiter((s.user_features.uid for s in samples), np.int64, B)
    profile = np.fromiter((s.user_features.profile_bucket for s in samples), np.int64, B)
    cand = np.fromiter((s.candidate.item_id for s in samples), np.int64, B)
    label = np.fromiter((s.label for s in samples), np.float64, B)
    if check:
        _check_ids("uid", uid, cfg.n_users)
        _check_ids("profile", profile, cfg.n_profiles)
        _check_ids("item", cand, cfg.vocab)
    return Batch(items, actions, dt, n.astype(np.int32), uid.astype(np.int32), profile.astype(np.int32),
                 cand.astype(np.int32), label.astype(np.float32))


def check_batch(batch: Batch, cfg: ModelConfig) -> None:
    """Range checks on an already-tensorised host batch (real tokens only)."""
    items = np.asarray(batch.items)
    L = cfg.L
    n = np.asarray(batch.n_events)
    if items.shape[1] != L:
        raise ConfigError(f"batch has L={items.shape[1]}, config L={L}")
    if (n < 0).any() or (n > L).any():
        raise ConfigError("n_events must lie in [0, L]")
    real = np.arange(L)[None, :] >= (L - n)[:, None]
    _check_ids("item", np.asarray(batch.items)[real], cfg.vocab)
    _check_ids("action", np.asarray(batch.actions)[real], cfg.n_actions)
    if (np.asarray(batch.dt)[real] < 0).any():
        raise ConfigError("future event: negative time delta")
    _check_ids("uid", np.asarray(batch.uid), cfg.n_users)
    _check_ids("profile", np.asarray(batch.profile), cfg.n_profiles)
    _check_ids("item", np.asarray(batch.cand_item), cfg.vocab)


def synthetic_samples(cfg: ModelConfig, n: int, seed: int = 1, n_events: Optional[int] = None,
                      base_time: int = 1_700_000_000, gap=(30, 900)) -> list:
    """Synthetic behaviour samples drawn exactly as BASELINE.md §3.1 prescribes (one
    ``default_rng(seed)`` consumed sample after sample: L × (gap, item, action), uid, profile,
    candidate item, label).  Gaps default to ``GeneratorConfig.gap_min/gap_max``."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        t = base_time
        ne = cfg.L if n_events is None else n_events
        events = []
        for _ in range(ne):
            t += int(rng.integers(gap[0], gap[1]))
            item = int(rng.integers(cfg.vocab))
            act = int(rng.integers(cfg.n_actions))
            events.append(Event(item, act, t))
        uid = int(rng.integers(cfg.n_users))
        prof = int(rng.integers(cfg.n_profiles))
        cand = int(rng.integers(cfg.vocab))
        label = int(rng.integers(2))
        out.append(Sample(tuple(events), UserFeatures(uid, prof), Candidate(cand, t + 60), label))
    return out


def synthetic_batch(cfg: ModelConfig, B: int, seed: int = 1, min_events: Optional[int] = None) -> Batch:
    """Vectorised synthetic batch (same distributions as :func:`synthetic_samples`, not the
    same stream): full-length sequences unless ``min_events`` is given."""
    rng = np.random.default_rng(seed)
    L = cfg.L
    gaps = rng.integers(30, 900, size=(B, L)).astype(np.int64)
    # dt of event j = sum of gaps after it + 60 s (candidate = last event + 60)
    dt = np.cumsum(gaps[:, ::-1], axis=1)[:, ::-1] - gaps + 60
    items = rng.integers(0, cfg.vocab, size=(B, L)).astype(np.int32)
    actions = rng.integers(0, cfg.n_actions, size=(B, L)).astype(np.int32)
    if min_events is None:
        n_ev = np.full(B, L, np.int32)
    else:
        n_ev = rng.integers(min_events, L + 1, size=B).astype(np.int32)
    real = np.arange(L)[None, :] >= (L - n_ev)[:, None]
    items = np.where(real, items, 0).astype(np.int32)
    actions = np.where(real, actions, 0).astype(np.int32)
    dt = np.where(real, np.minimum(dt, INT32_MAX), 0).astype(np.int32)
    uid = rng.integers(0, cfg.n_users, size=B).astype(np.int32)
    prof = rng.integers(0, cfg.n_profiles, size=B).astype(np.int32)
    cand = rng.integers(0, cfg.vocab, size=B).astype(np.int32)
    label = rng.integers(0, 2, size=B).astype(np.float32)
    return Batch(items, actions, dt, n_ev, uid, prof, cand, label)
