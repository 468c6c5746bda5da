"""Data parallelism over ranks: batch sharded, parameters replicated, one
gradient allreduce per step.

The reference is single-process (``train`` loops over samples, pkg/src/longrec/model.py:555-562)
and its SPEC permits batch-level data parallelism with a deterministic reduction order
(SPEC.md:86,387).  Each rank computes d(mean over its shard)/dθ; the global-batch gradient is
the size-weighted mean of the shard gradients, i.e. allreduce(sum of n_r·g_r) / Σ n_r — for
equal shards simply allreduce(sum)/world.  With a fixed world size NCCL/gloo reduce in a fixed
order, so the step is deterministic.
"""
from __future__ import annotations

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
