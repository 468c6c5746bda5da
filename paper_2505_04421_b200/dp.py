"""Data parallelism over ranks: batch sharded, parameters replicated, gradients
reduced in two buckets, the first one overlapping the front-end backward.

The reference is single-process (``train`` loops over samples, pkg/src/longrec/model.py:555-562)
and its SPEC permits batch-level data parallelism.  Each rank computes
d(mean BCE over its shard)/dθ; the global-batch gradient is the size-weighted mean of the shard
gradients, Σ_r n_r·g_r / Σ_r n_r — for equal shards the plain average.

Overlap.  ``longer_grad_early_begin`` splits the flat fp32 gradient buffer (``params()`` order)
into the blocks / query bank / head range, final before the front-end backward starts, and the
tables / token MLP / InnerTrans range written by the front-end kernels at the very end.  The step
records an event at the split point (``longer_set_grad_event``); a communication stream waits on
it and reduces the early range while the fused front-end backward kernels run, the late range is
reduced on the compute stream after the call, and the compute stream joins the communication
stream before the optimizer.  Everything is stream-ordered, so the whole step (fwd + bwd + both
reductions + Adam) captures into one CUDA graph.

Reproducibility: the per-rank gradients are summed with fp32 atomics inside the library (split-K
weight-gradient epilogues, LayerNorm / bias column sums, the item-table scatter), so bits can
differ from run to run at the last place; the cross-rank reduction itself has a fixed order for a
fixed world size (NCCL ring / gloo), so ranks always agree with each other.
"""
from __future__ import annotations

import ctypes

from .inputs import Batch


def shard_bounds(n: int, rank: int, world: int):
    """Contiguous, balanced shard [lo, hi) of n samples for `rank` (sizes differ by ≤ 1)."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_batch(batch: Batch, rank: int, world: int) -> Batch:
    lo, hi = shard_bounds(batch.size, rank, world)
    return Batch(**{f: getattr(batch, f)[lo:hi] for f in Batch.FIELDS})


def allreduce_mean_grads(grad_flat, local_n: int, group=None):
    """In place: grad_flat ← Σ_r n_r·g_r / Σ_r n_r (works for unequal shards)."""
    import torch
    import torch.distributed as dist
    grad_flat.mul_(float(local_n))
    n = torch.tensor([float(local_n)], dtype=grad_flat.dtype, device=grad_flat.device)
    dist.all_reduce(grad_flat, group=group)
    dist.all_reduce(n, group=group)
    grad_flat.div_(n)
    return grad_flat


def allreduce_mean_loss(loss_value: float, local_n: int, device="cpu", group=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([loss_value * local_n, float(local_n)], dtype=torch.float64, device=device)
    dist.all_reduce(t, group=group)
    return float(t[0] / t[1])


class DataParallel:
    """The data-parallel training-step body over an initialised ``torch.distributed`` group.

    ``loss_backward(local_batch)`` runs ``LongerModel.loss_backward`` on this rank's shard and
    leaves the global-batch gradient in ``model.grad_flat`` on every rank (stream-ordered on the
    caller's stream: follow it with ``Adam.step()``).  ``global_batch`` is the total number of
    samples over all ranks (default: world × local, i.e. equal shards).
    """

    def __init__(self, model, group=None, overlap: bool = True):
        import torch
        import torch.distributed as dist
        from . import _lib
        self.model = model
        self.group = group
        self.world = dist.get_world_size(group)
        self.backend = str(dist.get_backend(group)).lower()
        begin = ctypes.c_int64()
        _lib.check(model._lib.longer_grad_early_begin(ctypes.byref(_lib.dims_of(model.cfg, 1)),
                                                      ctypes.byref(begin)))
        self.split = int(begin.value)
        self.overlap = overlap and self.world > 1
        self.comm = torch.cuda.Stream(model.device)
        self.event = torch.cuda.Event()

    def _reduce(self, view, scale):
        import torch.distributed as dist
        if scale is None:                     # equal shards over NCCL: the average in the reduction
            dist.all_reduce(view, op=dist.ReduceOp.AVG, group=self.group)
        else:                                 # n_r / N folded in before a plain sum
            view.mul_(scale)
            dist.all_reduce(view, group=self.group)

    def loss_backward(self, local_batch, global_batch=None, check=False):
        import torch
        model = self.model
        n_local = local_batch.size if hasattr(local_batch, "size") and not callable(local_batch.size) \
            else len(local_batch)
        if self.world == 1:
            return model.loss_backward(local_batch, check=check)
        N = global_batch if global_batch is not None else self.world * n_local
        if N == self.world * n_local:         # equal shards: an average (gloo has no AVG op)
            scale = None if "nccl" in self.backend else 1.0 / self.world
        else:
            scale = float(n_local) / float(N)
        g = model.grad_flat
        if self.overlap:
            model._lib.longer_set_grad_event(ctypes.c_void_p(self.event.cuda_event))
        try:
            loss = model.loss_backward(local_batch, check=check)
        finally:
            if self.overlap:
                model._lib.longer_set_grad_event(None)
        main = torch.cuda.current_stream(model.device)
        if self.overlap:
            # blocks / bank / head: reduced on the communication stream beside the front-end bwd
            self.comm.wait_event(self.event)
            with torch.cuda.stream(self.comm):
                self._reduce(g[self.split:], scale)
            self._reduce(g[:self.split], scale)
            main.wait_stream(self.comm)
        else:
            self._reduce(g, scale)
        return loss
