"""``LongerModel`` — the drop-in for ``longrec.LongRecModel`` on the B200 path.

Same constructor (``LongerModel(cfg, seed)``), same ``params()`` names/shapes/order and the
same initial weights (``params.init_params`` replays the reference RNG stream), same
``forward``/``score`` semantics and the same checkpoint format (``LRCKPT01``,
``pkg/src/longrec/model.py:381-427``).  The difference: a call takes a whole batch and runs it
through the sm_100a library (``include/longer.h``) in one stream-ordered call; there is no CPU
fallback.

Master parameters are one fp32 device buffer in ``params()`` order (views per name); gradients
live in a second buffer of the same layout.
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Union

import numpy as np

from . import _lib
from .config import ModelConfig
from .errors import ConfigError, EmbeddingLookupError, NumericalError
from .inputs import Batch, Sample, check_batch, tensorize
from .params import init_params, param_shapes

def _torch():
    import torch
    return torch


@dataclass
class ForwardTrace:
    """Detached copies of every stage of one sample's forward (``ForwardTrace``,
    pkg/src/longrec/model.py:129-143): ``h`` [L, d] token-MLP output (zero rows for pad events),
    ``merged`` [G, D], the query indices (-1 for the learnable bank) and grid positions,
    ``layers`` = the [q, D] output of the cross block and of each self block, ``head_input``
    [1, 4D + 2d] and ``p``."""

    h: np.ndarray
    merged: np.ndarray
    query_indices: np.ndarray
    query_positions: np.ndarray
    layers: list = field(default_factory=list)
    head_input: Optional[np.ndarray] = None
    p: float = 0.0

    def sequence_branch(self) -> list:
        """All candidate-independent activations: everything but the target row."""
        return [self.h, self.merged] + [a[:-1] for a in self.layers]


class LongerModel:
    """Long-sequence recommender transformer (LONGER) on B200.

    ``forward(batch)`` → probabilities ``[B]`` (device tensor);
    ``loss_backward(batch)`` → batch-mean BCE (float) and fills ``grad_flat`` / ``grads()``.
    ``batch`` may be a list of ``Sample``, a host ``Batch`` (numpy) or a device ``Batch``.
    """

    def __init__(self, cfg: ModelConfig, seed: int = 0, device: str = "cuda") -> None:
        torch = _torch()
        cfg.validate()
        if cfg.d % 8:
            raise ConfigError("the B200 path needs d % 8 == 0 (16-byte rows for TMA)")
        self.cfg = cfg
        self.device = torch.device(device)
        if self.device.type != "cuda":
            raise RuntimeError("LongerModel runs on a CUDA (sm_100a) device only")
        self._lib = _lib.load()
        self.shapes = param_shapes(cfg)
        init = init_params(cfg, seed)
        flat = np.concatenate([a.ravel() for a in init.values()]).astype(np.float32)
        n = ctypes.c_int64()
        _lib.check(self._lib.longer_param_count(ctypes.byref(_lib.dims_of(cfg, 1)), ctypes.byref(n)))
        if n.value != flat.size:
            raise RuntimeError(f"parameter layout mismatch: library {n.value}, host {flat.size}")
        self.flat = torch.from_numpy(flat).to(self.device)
        self.grad_flat = torch.zeros_like(self.flat)
        self._views = self._make_views(self.flat)
        self._gviews = self._make_views(self.grad_flat)
        self.param_version = 0
        self._ws = {}
        self._probs = {}
        self._loss = torch.zeros(1, dtype=torch.float32, device=self.device)

    # ------------------------------------------------------------------ parameters
    def _make_views(self, buf):
        out, off = {}, 0
        for name, shape in self.shapes.items():
            size = int(np.prod(shape))
            out[name] = buf[off:off + size].view(*shape)
            off += size
        return out

    def params(self):
        """[(name, fp32 device tensor)] in reference order (pkg/src/longrec/model.py:252-263)."""
        return list(self._views.items())

    def grads(self):
        return list(self._gviews.items())

    def param_count(self) -> int:
        return int(self.flat.numel())

    def load_params(self, named) -> None:
        """Copy weights by name (e.g. from a reference ``LongRecModel.params()``)."""
        torch = _torch()
        for name, value in (named.items() if isinstance(named, dict) else named):
            data = getattr(value, "data", value)
            arr = np.asarray(data, dtype=np.float32)
            if name not in self._views:
                raise ConfigError(f"unknown parameter {name!r}")
            if tuple(arr.shape) != tuple(self._views[name].shape):
                raise ConfigError(f"parameter {name!r} shape {arr.shape} != {tuple(self._views[name].shape)}")
            self._views[name].copy_(torch.from_numpy(arr))
        self.param_version += 1

    def fingerprint(self) -> str:
        """sha256(config, param_version) (pkg/src/longrec/model.py:268-271)."""
        payload = json.dumps(self.cfg.to_dict(), sort_keys=True)
        return hashlib.sha256(f"{payload}|v{self.param_version}".encode()).hexdigest()[:16]

    # ------------------------------------------------------------------ batches
    def to_device_batch(self, batch: Union[Batch, Sequence[Sample]]) -> Batch:
        torch = _torch()
        if not isinstance(batch, Batch):
            batch = tensorize(list(batch), self.cfg)
        elif isinstance(batch.items, np.ndarray):
            check_batch(batch, self.cfg)
        if isinstance(batch.items, np.ndarray) or batch.items.device != self.device:
            batch = batch.to(self.device)
        return batch

    def _struct(self, b: Batch) -> _lib.LongerBatch:
        return _lib.LongerBatch(*[int(getattr(b, f).data_ptr()) for f in Batch.FIELDS])

    def _workspace(self, B: int):
        torch = _torch()
        if B not in self._ws:
            nbytes = ctypes.c_size_t()
            _lib.check(self._lib.longer_workspace_bytes(ctypes.byref(_lib.dims_of(self.cfg, B)), ctypes.byref(nbytes)))
            self._ws[B] = torch.zeros(nbytes.value + 256, dtype=torch.uint8, device=self.device)
            self._probs[B] = torch.zeros(B, dtype=torch.float32, device=self.device)
        ws = self._ws[B]
        base = (ws.data_ptr() + 255) & ~255
        return base, ws.numel() - (base - ws.data_ptr())

    def _stream(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def read_status(self, B: int) -> None:
        """Raise the reference error for device-detected bad inputs (ids / time deltas)."""
        base, _ = self._workspace(B)
        flags = ctypes.c_int32()
        _lib.check(self._lib.longer_read_status(ctypes.c_void_p(base), ctypes.byref(flags), self._stream()))
        if flags.value & 1:
            raise EmbeddingLookupError("an id fell outside its embedding table")
        if flags.value & 2:
            raise ConfigError("future event: negative time delta")

    # ------------------------------------------------------------------ compute
    def forward(self, batch, sync_check: bool = False):
        """Probabilities [B] (a new device tensor) for a batch (``forward_tensor`` + sigmoid,
        model.py:307-377).  A single ``Sample`` gives ``(p, ForwardTrace)`` like the reference's
        ``LongRecModel.forward(sample)`` (model.py:365-372)."""
        if isinstance(batch, Sample):
            p, traces = self.forward_traces([batch])
            return float(p[0]), traces[0]
        b = self.to_device_batch(batch)
        B = b.size
        base, nbytes = self._workspace(B)
        probs = self._probs[B]
        self._fwd_gen = getattr(self, "_fwd_gen", 0) + 1
        rc = self._lib.longer_forward(ctypes.byref(_lib.dims_of(self.cfg, B)), ctypes.c_void_p(self.flat.data_ptr()),
                                      ctypes.byref(self._struct(b)), ctypes.c_void_p(base), nbytes,
                                      ctypes.c_void_p(probs.data_ptr()), self._stream())
        _lib.check(rc)
        if sync_check:
            self.read_status(B)
        return probs.clone()

    def forward_traces(self, batch):
        """(probabilities [B] as numpy, [ForwardTrace per sample]): the forward with every row of
        every layer kept (``longer_forward_trace``), copied to the host."""
        torch = _torch()
        b = self.to_device_batch(batch)
        B = b.size
        base, nbytes = self._workspace(B)
        probs = self._probs[B]
        self._fwd_gen = getattr(self, "_fwd_gen", 0) + 1
        tr = _lib.LongerTrace()
        _lib.check(self._lib.longer_forward_trace(
            ctypes.byref(_lib.dims_of(self.cfg, B)), ctypes.c_void_p(self.flat.data_ptr()),
            ctypes.byref(self._struct(b)), ctypes.c_void_p(base), nbytes, ctypes.c_void_p(probs.data_ptr()),
            ctypes.byref(tr), self._stream()))
        self.read_status(B)
        ws = self._ws[B]
        cfg = self.cfg

        def view(ptr, shape, dtype=torch.float32):
            n = int(np.prod(shape))
            off = int(ptr) - ws.data_ptr()
            esz = torch.tensor([], dtype=dtype).element_size()
            return ws[off:off + n * esz].view(dtype).view(*shape).cpu().numpy()

        d, D, Lp, G, q = cfg.d, cfg.D, tr.Lp, tr.G, tr.q
        h = view(tr.h, (B, Lp, d))[:, Lp - cfg.L:].astype(np.float64)
        merged = view(tr.merged, (B, G, D)).astype(np.float64)
        layers = [view(tr.layers[i], (B, q, D)).astype(np.float64) for i in range(tr.n_layers)]
        head_in = view(tr.head_input, (B, tr.head_width)).astype(np.float64)
        k, K = cfg.k, cfg.K
        if cfg.query_strategy == "learnable":
            qidx = np.full((B, k), -1, np.int64)
            qpos_seq = np.full((B, k), (G - 1) * K + K - 1, np.int64)
        else:
            if tr.query_groups:
                qidx = view(tr.query_groups, (B, k), torch.int32).astype(np.int64)
            else:
                qidx = np.broadcast_to(np.arange(G - k, G, dtype=np.int64), (B, k)).copy()
            qpos_seq = qidx * K + K - 1
        qpos = np.concatenate([qpos_seq, np.zeros((B, cfg.m), np.int64)], axis=1)
        p = probs.cpu().numpy().astype(np.float64)
        traces = [ForwardTrace(h=h[i], merged=merged[i], query_indices=qidx[i], query_positions=qpos[i],
                               layers=[a[i] for a in layers], head_input=head_in[i:i + 1], p=float(p[i]))
                  for i in range(B)]
        return p, traces

    def vjp(self, batch, probs, dprobs):
        """(dprobs/dparams)ᵀ·dprobs into ``grad_flat`` (overwritten) for the batch the most recent
        ``forward`` ran on (its activations are still in the workspace); returns ``grad_flat``."""
        torch = _torch()
        b = self.to_device_batch(batch)
        B = b.size
        base, nbytes = self._workspace(B)
        dprobs = dprobs.to(device=self.device, dtype=torch.float32).contiguous()
        probs = probs.to(device=self.device, dtype=torch.float32).contiguous()
        _lib.check(self._lib.longer_backward(
            ctypes.byref(_lib.dims_of(self.cfg, B)), ctypes.c_void_p(self.flat.data_ptr()),
            ctypes.byref(self._struct(b)), ctypes.c_void_p(base), nbytes, ctypes.c_void_p(probs.data_ptr()),
            ctypes.c_void_p(dprobs.data_ptr()), ctypes.c_void_p(self.grad_flat.data_ptr()), self._stream()))
        return self.grad_flat

    def autograd_params(self):
        """A leaf tensor aliasing the flat fp32 master parameters, for ``LongerFunction``: after
        ``loss.backward()`` its ``.grad`` holds d(loss)/d(params) in ``params()`` order."""
        if getattr(self, "_leaf", None) is None:
            self._leaf = self.flat.detach().requires_grad_(True)
        return self._leaf

    def probs(self, batch):
        """Differentiable ``[B]`` probabilities (``torch.autograd`` bridge)."""
        b = self.to_device_batch(batch)
        return LongerFunction.apply(self.autograd_params(), self, b)

    def score(self, sample: Sample) -> float:
        """``LongRecModel.score`` (model.py:374-377)."""
        return float(self.forward([sample], sync_check=True)[0].item())

    def loss_backward(self, batch, check: Union[bool, str] = True):
        """Train-step body (model.py:555-567): grads ← d(mean BCE)/dparams.

        ``check=True``: the status flags and the loss come back in one D2H copy and one sync; a
        non-finite loss raises ``NumericalError`` exactly like ``train`` (model.py:563-566), a bad
        id ``EmbeddingLookupError``.  Returns the loss as a float.
        ``check="async"``: the same copy is queued to pinned host memory without a sync and
        inspected by later calls (``poll_checks``), so an error surfaces one or more steps late;
        returns the device loss tensor.  ``check=False``: no check, device loss tensor."""
        b = self.to_device_batch(batch)
        B = b.size
        base, nbytes = self._workspace(B)
        probs = self._probs[B]
        self._fwd_gen = getattr(self, "_fwd_gen", 0) + 1
        rc = self._lib.longer_forward_backward(
            ctypes.byref(_lib.dims_of(self.cfg, B)), ctypes.c_void_p(self.flat.data_ptr()),
            ctypes.byref(self._struct(b)), ctypes.c_void_p(base), nbytes, ctypes.c_void_p(probs.data_ptr()),
            ctypes.c_void_p(self._loss.data_ptr()), ctypes.c_void_p(self.grad_flat.data_ptr()), self._stream())
        _lib.check(rc)
        if not check:
            return self._loss
        slot = self._queue_check(B)
        if check == "async":
            self.poll_checks(block=False)
            return self._loss
        return self.poll_checks(block=True, until=slot)

    # ------------------------------------------------------------------ deferred input / loss checks
    def _queue_check(self, B: int):
        """[status flags, loss] → a pinned host slot (one D2H each, no sync); status reset."""
        torch = _torch()
        if not hasattr(self, "_chk_free"):
            from collections import deque
            self._chk_free = [torch.zeros(2, dtype=torch.int32).pin_memory() for _ in range(4)]
            self._chk_pending = deque()
        if not self._chk_free:                                 # ring full: retire the oldest
            self.poll_checks(block=True, until=self._chk_pending[0])
        host = self._chk_free.pop()
        base, _ = self._workspace(B)
        ws = self._ws[B]
        status = ws[base - ws.data_ptr():base - ws.data_ptr() + 4].view(torch.int32)
        host[0:1].copy_(status, non_blocking=True)
        status.zero_()
        host[1:2].copy_(self._loss.view(torch.int32), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        slot = (host, ev)
        self._chk_pending.append(slot)
        return slot

    def poll_checks(self, block: bool = False, until=None):
        """Inspect queued checks in order (waiting for them with ``block``, up to ``until``);
        raises the reference error of the first bad one.  Returns the last inspected loss."""
        value = None
        pend = getattr(self, "_chk_pending", None)
        while pend:
            host, ev = pend[0]
            if not block and not ev.query():
                break
            ev.synchronize()
            pend.popleft()
            flags = int(host[0])
            value = float(host[1:2].view(_torch().float32)[0])
            self._chk_free.append(host)
            if flags & 1:
                raise EmbeddingLookupError("an id fell outside its embedding table")
            if flags & 2:
                raise ConfigError("future event: negative time delta")
            if not math.isfinite(value):
                raise NumericalError("non-finite loss")
            if until is not None and (host, ev) is until:
                break
        return value

    # ------------------------------------------------------------------ checkpoints
    def save(self, path: str) -> None:
        """``LRCKPT01`` (model.py:381-406), loadable by ``longrec.LongRecModel.load``."""
        from .checkpoint import write_checkpoint
        write_checkpoint(path, self.cfg, [(n, v.detach().double().cpu().numpy()) for n, v in self.params()],
                         self.param_version)

    @classmethod
    def load(cls, path: str, device: str = "cuda") -> "LongerModel":
        """Read a reference (or our) ``LRCKPT01`` checkpoint (model.py:408-427)."""
        from .checkpoint import read_checkpoint
        cfg, named, version = read_checkpoint(path)
        model = cls(cfg, seed=0, device=device)
        model.load_params(named)
        model.param_version = version
        return model


def _autograd_base():
    import torch
    return torch.autograd.Function


class LongerFunction(_autograd_base()):
    """``probs = LongerFunction.apply(flat_params, model, batch)``: the LONGER forward as a
    ``torch.autograd.Function``.  Forward = ``longer_forward``; backward = ``longer_backward``, the
    vector-Jacobian product against the activations the forward left in the model's workspace —
    so a forward must be followed by its backward before the next forward of the same batch size
    on the same model (checked)."""

    @staticmethod
    def forward(ctx, flat, model, batch):
        probs = model.forward(batch).clone()
        ctx.model, ctx.batch, ctx.gen = model, batch, model._fwd_gen
        ctx.save_for_backward(probs)
        return probs

    @staticmethod
    def backward(ctx, dprobs):
        model = ctx.model
        if getattr(model, "_fwd_gen", None) != ctx.gen:
            raise RuntimeError("another LongerModel forward ran since this one; its activations are gone")
        (probs,) = ctx.saved_tensors
        grads = model.vjp(ctx.batch, probs, dprobs).clone()
        return grads, None, None


class Adam:
    """Adam with the reference's fixed hyper-parameters (model.py:453-482) on the flat buffers,
    one fused sm_100a kernel per step."""

    def __init__(self, model: LongerModel, lr: float) -> None:
        torch = _torch()
        self.model = model
        self.lr = float(lr)
        self.t = 0
        self.m = torch.zeros_like(model.flat)
        self.v = torch.zeros_like(model.flat)

    def step(self) -> None:
        self.t += 1
        mdl = self.model
        _lib.check(mdl._lib.longer_adam_step(
            ctypes.c_void_p(mdl.flat.data_ptr()), ctypes.c_void_p(mdl.grad_flat.data_ptr()),
            ctypes.c_void_p(self.m.data_ptr()), ctypes.c_void_p(self.v.data_ptr()), mdl.flat.numel(),
            self.lr, self.t, mdl._stream()))
        mdl.param_version += 1
