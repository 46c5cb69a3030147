"""Slice (path) sharding across GPUs -- the cut/slice driver's multi-GPU leg.

The amplitude is a sum over independent contraction paths
(rq/contraction_plan.py:1-34).  The reference walks them sequentially in
one process (rq/amplitude_engine.py:123, batch accumulation :153-157); here
the lexicographically sorted path list is cut into CONTIGUOUS chunks, one
per rank of a process group (one process per GPU), so each rank keeps the
`reuse=outer` intermediates of its own loop prefix, and the partial
amplitudes are summed with ONE all-reduce at the end.  The payload is a few
hundred bytes to a few KB (complex64 amplitudes as float32 pairs):
latency-bound, so one collective per call is the whole communication cost.

Sharding is strictly opt-in: `group=None` (the default everywhere) means
this process walks every path and nothing is reduced, whether or not
torch.distributed is initialised (bit-string sharding across ranks, for
example, must not sum amplitudes of different bit-strings).  Pass a
process group -- `torch.distributed.group.WORLD` for all ranks -- to shard
the paths over its ranks.

The all-reduce of device buffers on an NCCL group goes through the
library's own C ABI (`qf_nccl_init` / `qf_allreduce_c64`,
include/qflex_b200.h): the communicator is created once per (group,
device) from a unique id broadcast over the group, and the reduction is
enqueued on the caller's stream.  Other backends (gloo in the multi-process
CPU tests, or gloo on CUDA tensors) use torch.distributed.all_reduce.
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


def _active(group) -> bool:
    """True when `group` is a process group with more than one rank."""
    if group is None:
        return False
    if dist is None or not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("a slice group was given but torch.distributed is not initialised")
    return dist.get_world_size(group) > 1


def current_shard(group=None) -> SliceShard:
    """This process's shard of the path list: (0, 1) unless `group` is a
    process group, then (rank, size) within it."""
    if group is None:
        return SliceShard(0, 1)
    if dist is None or not dist.is_initialized():
        raise RuntimeError("a slice group was given but torch.distributed is not initialised")
    return SliceShard(dist.get_rank(group), dist.get_world_size(group))


_NATIVE: dict = {}        # (id(group), device index) -> library communicator handle
_native_enabled = True


def set_native_collective(enabled: bool) -> bool:
    """Use the library's NCCL all-reduce for device buffers on NCCL groups
    (default) or torch.distributed's; returns the previous setting."""
    global _native_enabled
    prev, _native_enabled = _native_enabled, bool(enabled)
    return prev


def _backend(group) -> str:
    try:
        return str(dist.get_backend(group)).lower()
    except Exception:  # pragma: no cover - backend query unsupported
        return ""


def native_comm(group, device) -> int:
    """The library communicator of (group, device), created on first use:
    rank 0 of the group draws an NCCL unique id (qf_nccl_unique_id), it is
    broadcast over the group, and every rank joins with qf_nccl_init."""
    from . import _lib
    dev = device.index if hasattr(device, "index") else int(device)
    key = (id(group), dev)
    h = _NATIVE.get(key)
    if h is not None:
        return h
    uid = _lib.nccl_unique_id() if dist.get_rank(group) == 0 else None
    box = [uid]
    src = dist.get_global_rank(group, 0) if group is not dist.group.WORLD else 0
    dist.broadcast_object_list(box, src=src, group=group)
    h = _lib.nccl_init(box[0], dist.get_world_size(group), dist.get_rank(group), dev)
    _NATIVE[key] = h
    return h


def reduce_partials(buf, group=None):
    """In-place sum of a complex (or real) buffer over the group's ranks;
    a no-op for group=None or a one-rank group.  Complex buffers travel as
    float pairs (NCCL has no complex type)."""
    if not _active(group):
        return buf
    if (_native_enabled and buf.is_cuda and buf.dtype == torch.complex64
            and _backend(group) == "nccl"):
        from . import _lib
        h = native_comm(group, buf.device)
        with torch.cuda.device(buf.device):
            _lib.allreduce_c64(h, buf, buf.numel())
        return buf
    view = torch.view_as_real(buf) if buf.is_complex() else buf
    dist.all_reduce(view, op=dist.ReduceOp.SUM, group=group)
    return buf


def reduce_int(value: int, group=None, device=None) -> int:
    """Sum an integer counter (e.g. executed flops) over the group."""
    if not _active(group):
        return int(value)
    t = torch.tensor([int(value)], dtype=torch.int64,
                     device=device if _backend(group) == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())
