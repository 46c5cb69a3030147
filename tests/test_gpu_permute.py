"""K1 permutation on the B200: bit-exact against the oracle (numpy
transpose, itself pinned to the reference's permute_fast bytes)."""

from __future__ import annotations

import hashlib
import os
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


# ---------------------------------------------------------------------------
# config 3 exactly as benchmarked: bench.config3_cases (64 seeded perms per
# size), every permutation byte-compared against the C oracle
# (oracle/permute_ref.c, the reference's permute_naive restated), with the
# bench's input values


def _host_ram_bytes() -> int:
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):  # pragma: no cover
        return 0


def _byte_compare_config3(log2n: int, count: int, which=None):
    from bench import config3_cases
    from oracle import permute_oracle as P
    n = 1 << log2n
    g = torch.Generator(device="cuda").manual_seed(log2n)
    src = torch.randn(n, dtype=torch.complex64, device="cuda", generator=g)
    dst = torch.empty_like(src)
    src_h = src.cpu().numpy()
    got_h = torch.empty(n, dtype=torch.complex64).pin_memory()
    want = np.empty(n, dtype=np.complex64)
    cases = config3_cases(log2n, 64, seed=log2n)
    picks = range(len(cases)) if which is None else which
    done = 0
    for i in list(picks)[:count]:
        dims, perm = cases[i]
        tc.permute_buffer(src, dims, perm, out=dst)
        got_h.copy_(dst)
        P.permute(src_h, dims, perm, out=want)
        assert got_h.numpy().tobytes() == want.tobytes(), (log2n, i, dims, perm)
        done += 1
    return done


def test_c_oracle_matches_numpy_oracle():
    from oracle import permute_oracle as P
    rng = np.random.default_rng(5)
    for _ in range(50):
        rank = int(rng.integers(1, 10))
        dims = [int(rng.integers(1, 5)) for _ in range(rank)]
        perm = [int(p) for p in rng.permutation(rank)]
        x = (rng.standard_normal(dims) + 1j * rng.standard_normal(dims)).astype(np.complex64)
        assert P.permute(x, dims, perm).tobytes() == O.permute_naive(x, perm).tobytes()


def test_config3_2pow24_all_64_byte_exact():
    assert _byte_compare_config3(24, 64) == 64


def test_config3_2pow28_all_64_byte_exact():
    if _host_ram_bytes() < 16 * 2 ** 30:
        pytest.skip("needs ~8 GiB of host RAM for the oracle buffers")
    assert _byte_compare_config3(28, 64) == 64


def test_config3_2pow30_byte_exact_sample():
    """8 of the 64 benchmarked 2^30 permutations (4 binary, 4 mixed), whole
    16 GiB tensors (8 GiB in + 8 GiB out) byte-compared."""
    if _host_ram_bytes() < 48 * 2 ** 30:
        pytest.skip("needs ~24 GiB of host RAM for the oracle buffers")
    assert _byte_compare_config3(30, 8, which=[0, 11, 22, 31, 32, 43, 54, 63]) == 8
