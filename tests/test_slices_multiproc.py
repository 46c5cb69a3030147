"""Multi-rank slice driver on CPU: world_size 2 over gloo (127.0.0.1).

Covers the host side of the multi-GPU path: contiguous path sharding
(every path exactly once, order preserved, reuse prefixes intact) and the
partial-amplitude all-reduce; the GPU run swaps gloo for NCCL."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_09599_b200 import slices
from paper_1811_09599_b200.contraction_plan import enumerate_paths


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # group=None never shards or reduces, even with the process group up
        assert slices.current_shard() == slices.SliceShard(0, 1)
        solo = torch.tensor([complex(rank + 1, 0)], dtype=torch.complex64)
        slices.reduce_partials(solo)
        assert solo.item() == complex(rank + 1, 0)
        assert slices.reduce_int(rank + 1) == rank + 1
        group = dist.group.WORLD
        shard = slices.current_shard(group)
        paths = enumerate_paths((8, 4), f=0.5, seed=3)
        mine = shard.take(paths)
        # partial "amplitudes": a deterministic function of the path
        part = torch.zeros(3, dtype=torch.complex64)
        for p in mine:
            part += torch.tensor([complex(p[0], p[1]), complex(1, 0), complex(p[0] * p[1], -1)],
                                 dtype=torch.complex64)
        slices.reduce_partials(part, group)
        flops = slices.reduce_int(len(mine) * 10, group)
        q.put((rank, mine, part.numpy(), flops))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 7, 16, 328):
        for world in (1, 2, 3, 8):
            spans = [slices.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(ValueError):
        slices.shard_range(4, 2, 2)


def test_two_rank_gloo_sum_equals_serial():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    paths = enumerate_paths((8, 4), f=0.5, seed=3)
    assert results[0][1] + results[1][1] == paths          # contiguous, complete, ordered
    want = np.zeros(3, np.complex64)
    for p in paths:
        want += np.array([complex(p[0], p[1]), 1, complex(p[0] * p[1], -1)], np.complex64)
    for _, _, part, flops in results:
        np.testing.assert_allclose(part, want, rtol=1e-6)
        assert flops == len(paths) * 10
