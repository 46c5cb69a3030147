"""The multi-GPU slice driver, engine level, on ONE GPU: two ranks on cuda:0
over gloo (gloo all-reduces CUDA tensors), each walking a contiguous half of
the path list of `AmplitudeEngine(group=WORLD)`; the all-reduced amplitudes
must equal the reference's golden values and the one-rank result.

This is the reference's sequential path loop (rq/amplitude_engine.py:123)
and batch accumulation (:153-157) sharded across ranks.  No kernel waits on
another rank's kernel (the only cross-rank step is the host-driven
all-reduce), so running both ranks on one device is sound.  The NCCL leg of
the same call (the library's qf_allreduce_c64) is covered with a one-rank
communicator in test_native_allreduce_one_rank."""

from __future__ import annotations

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT, golden_amps, rel_l2

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import paper_1811_09599_b200 as qf
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        with open(os.path.join(GOLDEN, "golden.json")) as fh:
            golden = json.load(fh)
        out = {}
        # config 2 (8 slices of one dim-8 cut -> 4 per rank), batched and single
        case = next(c for c in golden["amplitudes"] if c["name"] == "config2_c64")
        circ = qf.parse_circuit(golden["circuits"][case["circuit"]])
        plan = qf.parse_plan(golden["plans"][case["plan"]])
        eng = qf.AmplitudeEngine(circ, plan, group=dist.group.WORLD)
        got, stats = eng.amplitudes(case["in_bits"], case["out_bits"])
        single, sst = eng.amplitude(case["in_bits"], case["out_bits"][0])
        graph, _ = eng.amplitudes(case["in_bits"], case["out_bits"], graph=True)
        out["config2"] = (got, stats.paths_used, stats.flops, single, sst.flops, graph)
        # the open-qubit batch case (f < 1: a seeded subset of 65536 slices)
        bcase = next(c for c in golden["batches"] if c["name"] == "b70_t16_b64_f64")
        circ = qf.parse_circuit(golden["circuits"][bcase["circuit"]])
        plan = qf.parse_plan(golden["plans"][bcase["plan"]])
        eng = qf.AmplitudeEngine(circ, plan, group=dist.group.WORLD)
        b = eng.amplitude_batch(bcase["in_bits"], bcase["s_ab"], bcase["c_sites"], bcase["n_c"],
                                seed=bcase["seed"],
                                fidelity=qf.FidelitySpec(bcase["f"], bcase["fseed"]))
        out["batch"] = (b.amplitudes, b.stats.paths_used, b.stats.flops)
        # group=None with the process group up: the whole path list locally
        solo = qf.AmplitudeEngine(circ, plan)
        sb = solo.amplitude_batch(bcase["in_bits"], bcase["s_ab"], bcase["c_sites"],
                                  bcase["n_c"], seed=bcase["seed"],
                                  fidelity=qf.FidelitySpec(bcase["f"], bcase["fseed"]))
        out["solo"] = sb.amplitudes
        q.put((rank, out))
    except BaseException as exc:  # surface the failure to the parent
        q.put((rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def two_rank_results():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    return res


def test_two_ranks_config2_equal_golden(golden, two_rank_results):
    case = next(c for c in golden["amplitudes"] if c["name"] == "config2_c64")
    want = golden_amps(case)
    for rank, out in two_rank_results.items():
        got, used, flops, single, sflops, graph = out["config2"]
        assert rel_l2(got, want) < 1e-4, rank
        assert rel_l2(graph, want) < 1e-4, rank
        assert abs(single - want[0]) <= 1e-4 * abs(want[0]) + 1e-12, rank
        assert used == case["paths_used"]
        # flops are summed over the ranks: the whole path list once
        assert flops == case["flops"] and sflops == case["flops"]


def test_two_ranks_batch_equal_golden_and_one_rank(golden, two_rank_results):
    case = next(c for c in golden["batches"] if c["name"] == "b70_t16_b64_f64")
    want = golden_amps(case)
    r0 = two_rank_results[0]["batch"][0]
    for rank, out in two_rank_results.items():
        amps, used, flops = out["batch"]
        assert rel_l2(amps, want) < 1e-4, rank
        assert (used, flops) == (case["paths_used"], case["flops"])
        np.testing.assert_allclose(amps, r0, rtol=0, atol=0)   # both ranks hold the sum
        assert rel_l2(out["solo"], want) < 1e-4, rank          # group=None: unsharded
        assert rel_l2(out["solo"], amps) < 1e-5


def test_native_allreduce_one_rank():
    """qf_nccl_unique_id / qf_nccl_init / qf_allreduce_c64 through the C ABI
    with a one-rank communicator (the multi-rank NCCL run needs one GPU per
    rank): the sum over one rank is the identity, in place, on the stream."""
    from paper_1811_09599_b200 import _lib
    assert _lib.load().qf_nccl_available() == 1
    h = _lib.nccl_init(_lib.nccl_unique_id(), 1, 0, 0)
    x = torch.randn(1000, dtype=torch.complex64, device="cuda")
    y = x.clone()
    _lib.allreduce_c64(h, y, y.numel())
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    _lib.nccl_destroy(h)
    with pytest.raises(ValueError):
        _lib.allreduce_c64(h, y, y.numel())


def test_axpy_and_dot_c64():
    from paper_1811_09599_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(3 * 700, dtype=torch.complex64, device="cuda", generator=g)
    y = torch.randn(3 * 700, dtype=torch.complex64, device="cuda", generator=g)
    y0 = y.clone()
    _lib.axpy_c64(x, y, 0.5 - 2j)
    want = y0.cpu().numpy() + (0.5 - 2j) * x.cpu().numpy()
    assert rel_l2(y.cpu().numpy(), want) < 1e-6
    out = torch.empty(3, dtype=torch.complex64, device="cuda")
    _lib.dot_c64(x, y0, out, batch=3, n=700)
    xh, yh = x.cpu().numpy().reshape(3, 700), y0.cpu().numpy().reshape(3, 700)
    want = (xh.astype(np.complex128) * yh).sum(axis=1)
    assert rel_l2(out.cpu().numpy(), want) < 1e-5
