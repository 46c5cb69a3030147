"""Slice (path) sharding across GPUs -- the cut/slice driver's multi-GPU leg.

The amplitude is a sum over independent contraction paths
(rq/contraction_plan.py:1-34).  The reference walks them sequentially in
one process (rq/amplitude_engine.py:123); here the lexicographically
sorted path list is cut into CONTIGUOUS chunks, one per rank (one process
per GPU), so each rank keeps the `reuse=outer` intermediates of its own
loop prefix, and the partial amplitudes are summed with ONE all-reduce over
NCCL (NVLink/NVSwitch) at the end.  The payload is a few hundred bytes to a
few KB (complex64 amplitudes as float32 pairs): latency-bound, so one
collective per call is the whole communication cost.

The functions here are backend-agnostic (NCCL for GPU tensors, gloo for
CPU tensors in the multi-process CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Sequence

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None


@dataclass(frozen=True)
class SliceShard:
    rank: int
    world: int

    def range(self, n_paths: int) -> tuple:
        """[lo, hi) of this rank's contiguous share of n_paths paths."""
        return shard_range(n_paths, self.rank, self.world)

    def take(self, paths: Sequence) -> list:
        lo, hi = self.range(len(paths))
        return list(paths[lo:hi])


def shard_range(n: int, rank: int, world: int) -> tuple:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad shard rank={rank} world={world}")
    return (n * rank) // world, (n * (rank + 1)) // world


def current_shard(group=None) -> SliceShard:
    """The calling process's shard (world 1 when torch.distributed is off)."""
    if dist is None or not dist.is_available() or not dist.is_initialized():
        return SliceShard(0, 1)
    return SliceShard(dist.get_rank(group), dist.get_world_size(group))


def reduce_partials(buf, group=None):
    """In-place sum of a complex (or real) buffer over the group's ranks.
    Complex buffers travel as float pairs (NCCL has no complex type)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return buf
    view = torch.view_as_real(buf) if buf.is_complex() else buf
    dist.all_reduce(view, op=dist.ReduceOp.SUM, group=group)
    return buf


def reduce_int(value: int, group=None, device=None) -> int:
    """Sum an integer counter (e.g. executed flops) over the group."""
    if dist is None or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())
