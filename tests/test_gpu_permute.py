"""K1 permutation on the B200: bit-exact against the oracle (numpy
transpose, itself pinned to the reference's permute_fast bytes)."""

from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest
import torch

from oracle import rqc_oracle as O
from paper_1811_09599_b200 import tensor_core as tc

pytestmark = pytest.mark.gpu


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).reshape(-1)).cuda()


def _run(x, perm):
    out = tc.permute_buffer(_dev(x), x.shape, perm)
    torch.cuda.synchronize()
    return out[: x.size].cpu().numpy()


def test_golden_cases_byte_exact(golden_perm):
    for case in golden_perm["cases"]:
        g = np.random.default_rng(case["input_seed"])
        dims = case["dims"]
        x = (g.standard_normal(dims) + 1j * g.standard_normal(dims)).astype(np.complex64)
        got = _run(x, case["perm"])
        assert hashlib.sha256(got.tobytes()).hexdigest() == case["sha256"], case


def test_random_small_cases_c64_and_c128():
    rng = np.random.default_rng(91)
    for i in range(300):
        rank = int(rng.integers(1, 9))
        dims = [int(rng.integers(1, 6)) for _ in range(rank)]
        perm = [int(p) for p in rng.permutation(rank)]
        dt = np.complex64 if i % 3 else np.complex128
        x = (rng.standard_normal(dims) + 1j * rng.standard_normal(dims)).astype(dt)
        assert _run(x, perm).tobytes() == O.permute_naive(x, perm).tobytes(), (dims, perm)


def _config3_case(rng, log2n, binary):
    if binary:
        dims = [2] * log2n
    else:
        bits = []
        while sum(bits) < log2n:
            b = int(rng.integers(1, 5))
            bits.append(min(b, log2n - sum(bits)))
        if len(bits) < 10:
            return _config3_case(rng, log2n, binary)
        dims = [1 << b for b in bits]
    perm = [int(p) for p in rng.permutation(len(dims))]
    return dims, perm


@pytest.mark.parametrize("binary", [True, False])
def test_config3_2pow24_byte_exact(binary):
    rng = np.random.Generator(np.random.PCG64(24 + binary))
    for _ in range(8):
        dims, perm = _config3_case(rng, 24, binary)
        x = (rng.standard_normal(1 << 24, dtype=np.float32)
             + 1j * rng.standard_normal(1 << 24, dtype=np.float32)).astype(np.complex64)
        x = x.reshape(dims)
        assert _run(x, perm).tobytes() == O.permute_naive(x, perm).tobytes()


def test_config3_2pow28_roundtrip_property():
    """Size-independent property at 2^28: permute then inverse-permute is
    the identity, and a permuted checksum matches the oracle on a sample."""
    rng = np.random.Generator(np.random.PCG64(28))
    dims, perm = _config3_case(rng, 28, True)
    n = 1 << 28
    src = torch.randn(n, dtype=torch.complex64, device="cuda")
    mid = tc.permute_buffer(src, dims, perm)
    inv = [perm.index(i) for i in range(len(perm))]
    back = tc.permute_buffer(mid, [dims[p] for p in perm], inv)
    torch.cuda.synchronize()
    assert torch.equal(back[:n], src)
    # spot check 4096 output positions against the index arithmetic
    out_dims = [dims[p] for p in perm]
    idx = rng.integers(0, n, size=4096)
    strides = [math.prod(dims[i + 1:]) for i in range(len(dims))]
    src_idx = np.zeros_like(idx)
    rem = idx.copy()
    for j in range(len(out_dims) - 1, -1, -1):
        src_idx += (rem % out_dims[j]) * strides[perm[j]]
        rem //= out_dims[j]
    got = mid[torch.from_numpy(idx).cuda()].cpu().numpy()
    want = src[torch.from_numpy(src_idx).cuda()].cpu().numpy()
    assert got.tobytes() == want.tobytes()


def test_identity_and_rank0_and_empty():
    x = np.arange(12, dtype=np.complex64).reshape(3, 4)
    assert _run(x, [0, 1]).tobytes() == x.tobytes()
    s = np.array(5 + 1j, dtype=np.complex64)
    assert tc.permute_fast(s.reshape(()), tc.plan_permutation((), ())).tobytes() == s.tobytes()
    empty = torch.zeros(1, dtype=torch.complex64, device="cuda")
    tc.permute_buffer(empty, (0, 3), (1, 0))   # zero elements: no-op, no error
    torch.cuda.synchronize()


def test_reference_api_shims():
    rng = np.random.default_rng(3)
    x = (rng.standard_normal((2,) * 7) + 0j).astype(np.complex64)
    perm = [2, 5, 4, 0, 3, 6, 1]
    plan = tc.plan_permutation([2] * 7, perm, mu=2, nu=4)
    assert tc.permute_fast(x, plan).tobytes() == O.permute_naive(x, perm).tobytes()
    assert tc.permute_naive(x, perm).tobytes() == O.permute_naive(x, perm).tobytes()
    with pytest.raises(ValueError):
        tc.plan_permutation([2, 2], [0, 0])


def test_benchmark_permute_schema_and_perms():
    rows = tc.benchmark_permute(rank=16, gammas=range(5, 7), repeats=3)
    assert [r["op"] for r in rows] == ["lmove", "rmove", "naive"] * 2
    assert all(r["median_ns"] > 0 and r["p10_ns"] <= r["p90_ns"] for r in rows)
    csv = tc.benchmark_csv(rows)
    assert csv.splitlines()[0] == "op,rank,gamma,threads,median_ns,p10_ns,p90_ns"
    assert len(csv.splitlines()) == 7
