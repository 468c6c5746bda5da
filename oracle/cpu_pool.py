"""Multi-process CPU training step of the oracle port — TEST INFRASTRUCTURE (bench.py's reference
arm and its ``cpu_baseline``), never imported by the product package.

The reference (``longrec``) trains in one process (``train``, pkg/src/longrec/model.py:534-577);
SPEC.md:86 permits batch-level data parallelism, so the fastest faithful CPU path on an n-core
host is n single-threaded worker processes (BLAS threads = 1), each running the float64
forward + backward of its shard of the batch (``longer_oracle.forward_backward``, pinned to the
reference's own outputs by tests/test_oracle.py), the parent summing the size-weighted shard
gradients and applying Adam (model.py:555-569, 453-482) — the same step the GPU arm times.
"""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

_STATE = {}


def _init(cfg_kw, seed):
    from paper_2505_04421_b200 import ModelConfig, init_params
    cfg = ModelConfig(**cfg_kw).validate()
    _STATE["cfg"] = cfg
    _STATE["P"] = init_params(cfg, seed)


def _shard(task):
    from oracle import longer_oracle as O
    flat, batch = task
    P, cfg, off = _STATE["P"], _STATE["cfg"], 0
    for name, a in P.items():                 # this step's parameters
        P[name] = flat[off:off + a.size].reshape(a.shape)
        off += a.size
    n = len(batch["label"])
    _, loss, grads = O.forward_backward(P, cfg, batch)
    return n, loss * n, np.concatenate([grads[k].ravel() for k in P]) * n


class CpuPool:
    """``workers`` single-threaded processes; ``step(batch)`` = one data-parallel training step
    (fwd + bwd on shards, gradient sum, Adam) of the float64 oracle; returns the batch loss."""

    def __init__(self, cfg, workers=None, seed=0, lr=None):
        from paper_2505_04421_b200 import init_params
        self.cfg = cfg
        self.workers = workers or os.cpu_count() or 1
        saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")}
        os.environ.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1")
        try:
            ctx = mp.get_context("spawn")
            self.pool = ctx.Pool(self.workers, initializer=_init, initargs=(cfg.to_dict(), seed))
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        P = init_params(cfg, seed)
        self.names = list(P)
        self.flat = np.concatenate([a.ravel() for a in P.values()]).astype(np.float64)
        self.m = np.zeros_like(self.flat)
        self.v = np.zeros_like(self.flat)
        self.t = 0
        self.lr = cfg.lr if lr is None else lr

    def step(self, batch: dict) -> float:
        from oracle import longer_oracle as O
        B = len(batch["label"])
        bounds = np.linspace(0, B, min(self.workers, B) + 1).astype(int)
        shards = [{k: v[lo:hi] for k, v in batch.items()} for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]
        out = self.pool.map(_shard, [(self.flat, s) for s in shards], chunksize=1)
        n = sum(o[0] for o in out)
        loss = sum(o[1] for o in out) / n
        grad = sum(o[2] for o in out) / n
        self.t += 1
        O.adam_step(self.flat, grad, self.m, self.v, self.t, self.lr)
        return float(loss)

    def close(self):
        self.pool.terminate()
        self.pool.join()


def cpu_model_name() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
