"""K2/K3 complex GEMM on the B200 against a float64 numpy reference
(tolerance: relative Frobenius 1e-5 for complex64, 1e-12 for complex128)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_1811_09599_b200 import _lib
from paper_1811_09599_b200 import tensor_core as tc

pytestmark = pytest.mark.gpu


def _rand(rng, shape, dt):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(dt)


def _gemm(batch, M, N, K, opA, opB, dt, mode=None, alpha=1.0, beta=0.0, seed=0):
    rng = np.random.default_rng(seed)
    A = _rand(rng, (batch, M, K) if opA == 0 else (batch, K, M), dt)
    B = _rand(rng, (batch, K, N) if opB == 0 else (batch, N, K), dt)
    C0 = _rand(rng, (batch, M, N), dt)
    dA, dB = torch.from_numpy(A.reshape(-1)).cuda(), torch.from_numpy(B.reshape(-1)).cuda()
    dC = torch.from_numpy(C0.reshape(-1)).cuda()
    tc.gemm_buffer(batch, M, N, K, dA, opA, dB, opB, dC, alpha, beta, mode)
    torch.cuda.synchronize()
    a = A if opA == 0 else A.transpose(0, 2, 1)
    b = B if opB == 0 else B.transpose(0, 2, 1)
    want = alpha * np.matmul(a.astype(np.complex128), b.astype(np.complex128)) + beta * C0
    got = dC.cpu().numpy().reshape(batch, M, N)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


SHAPES = [(1, 64, 64, 64), (3, 100, 37, 70), (2, 4096, 64, 64), (1, 1, 1, 4096),
          (4, 1, 64, 20000), (1, 64, 1, 5000), (1, 257, 129, 33), (5, 7, 5, 3), (1, 8, 8, 0),
          (1, 512, 512, 256), (3, 1000, 1, 64), (2, 4096, 3, 100), (1, 77, 4, 33),
          (16, 4096, 1, 64), (2, 300, 2, 1000)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("ops", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_ffma_c64(shape, ops):
    assert _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_FFMA) < 1e-5


@pytest.mark.parametrize("shape", SHAPES[:6])
def test_zgemm_c128(shape):
    assert _gemm(*shape, 0, 1, np.complex128) < 1e-12


def test_alpha_beta():
    assert _gemm(2, 33, 65, 17, 0, 0, np.complex64, _lib.GEMM_FFMA, 0.5 - 1j, 1.0 + 0.5j) < 1e-5
    assert _gemm(1, 1, 3, 9000, 0, 0, np.complex64, _lib.GEMM_FFMA, 2.0, 1.0) < 1e-5


def test_contract_matches_einsum():
    rng = np.random.default_rng(3)
    a = tc.Tensor(("i", "j", "k"), _rand(rng, (4, 3, 2), np.complex64))
    b = tc.Tensor(("j", "k", "m"), _rand(rng, (3, 2, 5), np.complex64))
    out = tc.contract(a, b)
    ref = np.einsum("ijk,jkm->im", a.array, b.array)
    assert set(out.labels) == {"i", "m"}
    np.testing.assert_allclose(out.transpose_to(("i", "m")).array, ref, rtol=1e-5, atol=1e-6)
    v = tc.Tensor(("x",), np.array([1.0, 2.0], np.complex64))
    w = tc.Tensor(("y",), np.array([3.0, 5.0], np.complex64))
    np.testing.assert_allclose(tc.contract(v, w).transpose_to(("x", "y")).array,
                               [[3, 5], [6, 10]])
    s = tc.contract(tc.Tensor(("x",), np.arange(8, dtype=np.complex64)),
                    tc.Tensor(("x",), np.ones(8, np.complex64))).scalar()
    assert abs(s - 28) < 1e-5
    with pytest.raises(ValueError):
        tc.contract(tc.Tensor(("i", "j"), np.zeros((2, 3), np.complex64)),
                    tc.Tensor(("j", "k"), np.zeros((4, 2), np.complex64)))


def test_batched_contract_keeps_batch_label():
    rng = np.random.default_rng(4)
    A = _rand(rng, (6, 4, 3, 2), np.complex64)
    B = _rand(rng, (6, 2, 3, 5), np.complex64)
    a = tc.Tensor(("@b", "i", "j", "k"), A)
    b = tc.Tensor(("@b", "k", "j", "m"), B)
    out = tc.contract(a, b)
    assert out.labels[0] == "@b"
    ref = np.einsum("bijk,bkjm->bim", A, B)
    np.testing.assert_allclose(out.transpose_to(("@b", "i", "m")).array, ref, rtol=1e-5,
                               atol=1e-6)


TC_SHAPES = [(1, 128, 128, 8), (1, 128, 128, 64), (2, 256, 256, 40), (1, 300, 200, 77),
             (3, 4096, 64, 64), (1, 1000, 130, 1000), (4, 512, 64, 8), (1, 129, 257, 3),
             (1, 2048, 2048, 512)]

# short-K runs: B panels kept in the stage ring across consecutive tiles
# (k-block counts 1/2/4/8, ragged K and M, several N tiles per batch, runs
# that cross batch boundaries, runs of one tile)
SHORTK_SHAPES = [(2, 1024, 192, 32), (5, 1000, 64, 60), (64, 256, 64, 16), (256, 512, 64, 64),
                 (40, 640, 96, 8), (3, 2048, 128, 24), (7, 384, 64, 200),
                 # narrow N tiles (BN = 8 / 16 / 32, ragged columns)
                 (64, 512, 8, 64), (16, 1000, 8, 8), (8, 2048, 16, 40), (5, 700, 12, 64),
                 (9, 300, 5, 24), (4, 640, 32, 64), (3, 512, 24, 130)]


@pytest.fixture(params=[0, 10, 11, 12, 13, 19, 20, 21, 26, 31, 34],
                ids=["auto", "short-8warps", "short-16warps", "short-epilogue-warps",
                     "long-converter-fetch", "long-real-block", "short-tma", "short-tma-ring4",
                     "long-real-block-ck16", "long-gauss-ck32", "long-gauss-2stages"])
def tc_variant(request):
    lib = _lib.load()
    prev = lib.qf_tc3_set_variant(request.param)
    yield request.param
    lib.qf_tc3_set_variant(prev)


@pytest.mark.parametrize("shape", TC_SHAPES)
@pytest.mark.parametrize("ops", [(0, 0), (1, 1), (0, 1), (1, 0)])
def test_tcgen05_3xtf32_c64(shape, ops, tc_variant):
    """3xTF32 keeps ~fp32 accuracy: same 1e-5 bar as the FFMA kernel."""
    err = _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_TC3)
    assert err < 1e-5, err


@pytest.mark.parametrize("shape", SHORTK_SHAPES)
@pytest.mark.parametrize("ops", [(0, 0), (1, 1), (0, 1), (1, 0)])
@pytest.mark.parametrize("variant", [0, 10, 11, 12, 20],
                         ids=["auto", "8warps", "16warps", "epilogue-warps", "tma"])
def test_tcgen05_short_k_runs(shape, ops, variant):
    lib = _lib.load()
    prev = lib.qf_tc3_set_variant(variant)
    try:
        assert _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_TC3) < 1e-5
    finally:
        lib.qf_tc3_set_variant(prev)


@pytest.mark.parametrize("a_labels", [["@b", "p", "s", "q", "t"], ["@b", "s", "q", "t", "p"]],
                         ids=["k-innermost", "row-innermost"])
@pytest.mark.parametrize("variant", [10, 11, 12],
                         ids=["8warps", "16warps", "epilogue-warps"])
def test_gathered_short_k_many_tiles(a_labels, variant):
    """Gathered A through the short-K kernel with several M tiles per batch
    (row offsets prefetched a tile ahead, B reused across the run), for both
    fetch layouts: summed label innermost (lanes along k) and free label
    innermost (lane = row)."""
    rng = np.random.default_rng(7)
    dims = {"@b": 6, "p": 16, "s": 8, "q": 32, "t": 8}
    A = _rand(rng, tuple(dims[l] for l in a_labels), np.complex64)
    B = _rand(rng, (6, 8, 64, 8), np.complex64)          # @b t v s
    lib = _lib.load()
    prev = tc.set_gemm_mode("tc3")
    prev_v = lib.qf_tc3_set_variant(variant)
    try:
        out = tc.contract(tc.Tensor(a_labels, A), tc.Tensor(["@b", "t", "v", "s"], B))
        got = out.transpose_to(["@b", "p", "q", "v"]).array
    finally:
        tc.set_gemm_mode(prev)
        lib.qf_tc3_set_variant(prev_v)
    sub = {"@b": "z", "p": "p", "s": "s", "q": "q", "t": "t"}
    ref = np.einsum("".join(sub[l] for l in a_labels) + ",ztvs->zpqv", A.astype(np.complex128),
                    B.astype(np.complex128))
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("K", [1024, 4096, 32768])
@pytest.mark.parametrize("variant", [0, 13, 19, 26, 27, 30, 31, 34],
                         ids=["default", "converter-fetch", "real-block-ck4", "real-block-ck16",
                              "real-block-ck32", "gauss-ck16", "gauss-ck32", "gauss-2stages"])
def test_tcgen05_promoted_accuracy_at_long_k(K, variant):
    """Promotion keeps the long-K error near the FFMA kernel's (config-4
    GEMMs have K = 2^15)."""
    lib = _lib.load()
    prev = lib.qf_tc3_set_variant(variant)
    try:
        err = _gemm(1, 128, 64, K, 0, 0, np.complex64, mode=_lib.GEMM_TC3)
    finally:
        lib.qf_tc3_set_variant(prev)
    assert err < 5e-6, err


def test_tcgen05_alpha_beta(tc_variant):
    assert _gemm(2, 256, 128, 64, 0, 0, np.complex64, _lib.GEMM_TC3, 0.5 - 1j, 1.0 + 0.5j) < 1e-5


@pytest.mark.parametrize("shape", [(16, 1024, 128, 512), (64, 512, 64, 64), (64, 512, 16, 64),
                                   (3, 2048, 2048, 1024)])
@pytest.mark.parametrize("ab", [(0.5 - 1j, 0.0), (1.0, 0.5 + 0.25j), (1.0, 0.0)])
@pytest.mark.parametrize("ops", [(0, 0), (1, 1)])
def test_tcgen05_alpha_beta_multi_tile_runs(shape, ab, ops):
    """alpha/beta (per-element epilogue paths) with several tiles per CTA."""
    assert _gemm(*shape, *ops, np.complex64, _lib.GEMM_TC3, ab[0], ab[1]) < 1e-5


def test_tcgen05_matches_ffma_bitwise_scale():
    """Same inputs through both engines agree to ~fp32 rounding (the
    tensor-core engine promotes its fp32 partial every 512 k, whose
    truncating accumulation costs ~4e-6 relative)."""
    rng = np.random.default_rng(11)
    M, N, K = 512, 256, 1024
    A = _rand(rng, (M, K), np.complex64)
    B = _rand(rng, (K, N), np.complex64)
    outs = []
    for mode in (_lib.GEMM_FFMA, _lib.GEMM_TC3):
        C = torch.empty(M * N, dtype=torch.complex64, device="cuda")
        tc.gemm_buffer(1, M, N, K, torch.from_numpy(A.reshape(-1)).cuda(), 0,
                       torch.from_numpy(B.reshape(-1)).cuda(), 0, C, mode=mode)
        outs.append(C.cpu().numpy())
    assert np.linalg.norm(outs[0] - outs[1]) / np.linalg.norm(outs[0]) < 6e-6


@pytest.mark.parametrize("mode", ["auto", "ffma", "tc3"])
@pytest.mark.parametrize("case", range(5))
def test_gathered_a_contract_matches_permuted(mode, case):
    """Gathered-A GEMMs (operand permutation fused into the fetch) give the
    same contraction as permute-then-GEMM, for scattered shared labels."""
    rng = np.random.default_rng(100 + case)
    batch = [1, 4, 16, 2, 8][case]
    dims = {"p": 8, "q": 8, "r": 4, "s": 8, "t": 8, "u": 2, "v": 8}
    a_labels = ["@b", "p", "s", "q", "t", "r"][: 6] if case % 2 == 0 else ["@b", "s", "p", "t", "q", "r"]
    b_labels = ["@b", "t", "v", "s"] if case < 3 else ["@b", "s", "u", "t"]
    A = _rand(rng, [batch] + [dims[l] for l in a_labels[1:]], np.complex64)
    B = _rand(rng, [batch] + [dims[l] for l in b_labels[1:]], np.complex64)
    prev = qf_mode = tc.set_gemm_mode(mode)
    try:
        outs = []
        for gather in (True, False):
            tc.set_gather(gather)
            out = tc.contract(tc.Tensor(a_labels, A), tc.Tensor(b_labels, B))
            keep = [l for l in a_labels if l not in b_labels or l == "@b"] + \
                   [l for l in b_labels if l not in a_labels]
            outs.append(out.transpose_to(keep).array)
        sub = {"@b": "z", "p": "p", "q": "q", "r": "r", "s": "s", "t": "t", "u": "u", "v": "v"}
        spec = "".join(sub[l] for l in a_labels) + "," + "".join(sub[l] for l in b_labels) + "->" + \
            "".join(sub[l] for l in keep)
        ref = np.einsum(spec, A.astype(np.complex128), B.astype(np.complex128))
        for o in outs:
            assert np.linalg.norm(o - ref) / np.linalg.norm(ref) < 1e-5
    finally:
        tc.set_gather(True)
        tc.set_gemm_mode(prev)


@pytest.mark.parametrize("engine", [0, 1, 2, 3], ids=["auto", "smem", "rowblock", "rowstream"])
@pytest.mark.parametrize("shape", [(3, 4096, 8, 64), (2, 4096, 64, 8), (1, 32768, 8, 8),
                                   (4, 512, 512, 8), (2, 100, 13, 7), (1, 77, 3, 300),
                                   (5, 1000, 8, 64), (7, 333, 5, 24), (3, 64, 16, 32)])
@pytest.mark.parametrize("ops", [(0, 0), (1, 1), (0, 1)])
def test_small_kxn_engines(engine, shape, ops):
    lib = _lib.load()
    prev = lib.qf_small_engine(engine)
    try:
        assert _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_FFMA) < 1e-5
        assert _gemm(*shape[:3], shape[3], *ops, np.complex128) < 1e-12
    finally:
        lib.qf_small_engine(prev)


@pytest.mark.parametrize("mode", ["auto", "ffma", "tc3"])
@pytest.mark.parametrize("case", range(6))
def test_late_sliced_contract_matches_numpy(mode, case):
    """Late output slicing: a tensor with open `out` indices (anywhere in its
    layout, innermost included) contracted with a batched tensor -- the
    per-bit-string slice fused into the gathered GEMM fetch
    (qf_cgemm_c64_gather_boff) or materialised (qf_gather_rows) -- equals
    slicing first and contracting per bit-string."""
    rng = np.random.default_rng(300 + case)
    nb = [16, 64, 5, 33, 128, 8][case]
    dims = {"p": 8, "q": 8, "r": 4, "s": 8, "t": 8, "v": 16, "out0": 2, "out1": 2, "out2": 2}
    a_labels = [["p", "out0", "s", "q", "t", "out1"], ["out1", "s", "p", "t", "q", "r"],
                ["p", "s", "out0", "out2", "q", "t"], ["s", "p", "out0", "t", "out1", "q"],
                ["p", "q", "s", "t", "out2"], ["out0", "out1", "out2", "s", "t", "p"]][case]
    b_labels = ["@b", "t", "v", "s"]
    outs = [l for l in a_labels if l.startswith("out")]
    A = _rand(rng, [dims[l] for l in a_labels], np.complex64)
    B = _rand(rng, [nb] + [dims[l] for l in b_labels[1:]], np.complex64)
    bits = rng.integers(0, 2, size=(3, nb)).astype(np.int32)
    rows = {"out0": 0, "out1": 1, "out2": 2}
    late = tc.LateBits(torch.from_numpy(bits).cuda(), {l: rows[l] for l in outs})
    prev = tc.set_gemm_mode(mode)
    try:
        ta, tb = tc.Tensor(a_labels, A), tc.Tensor(b_labels, B)
        got = tc.contract_late(ta, tb, late)
        sliced = late.batch(ta)
        assert sliced.labels[0] == "@b" and not late.outs(sliced)
    finally:
        tc.set_gemm_mode(prev)
    rest = [l for l in a_labels if l not in outs]
    idx = tuple(bits[rows[l]] if l in outs else slice(None) for l in a_labels)
    # numpy advanced indexing: the batch axis lands first when the indexed
    # axes are not adjacent, else in place of the first one -- move it first
    As = A[idx]
    first = min(a_labels.index(l) for l in outs)
    adjacent = all(a_labels.index(o) - first == i for i, o in enumerate(outs))
    if adjacent and first > 0:
        As = np.moveaxis(As, first, 0)
    np.testing.assert_array_equal(sliced.array, As)
    keep = ["@b"] + [l for l in rest if l not in b_labels] + [l for l in b_labels[1:] if l not in rest]
    sub = {l: chr(ord("a") + i) for i, l in enumerate(["@b"] + list(dims))}
    spec = "".join(sub[l] for l in ["@b"] + rest) + "," + "".join(sub[l] for l in b_labels) + \
        "->" + "".join(sub[l] for l in keep)
    ref = np.einsum(spec, As.astype(np.complex128), B.astype(np.complex128))
    out = got.transpose_to(keep).array
    assert np.linalg.norm(out - ref) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("mode", ["auto", "ffma", "tc3"])
@pytest.mark.parametrize("case", range(4))
def test_late_open_contract_equals_plain(mode, case):
    """Two operands with open outputs and no batch axis: the smaller one's
    outputs become the GEMM batch (big operand broadcast) -- same tensor as
    the plain contraction, outputs moved to the front."""
    rng = np.random.default_rng(400 + case)
    dims = {"p": 8, "q": 8, "s": 8, "t": 8, "v": 8, "out0": 2, "out1": 2, "out2": 2}
    a_labels = [["p", "out0", "s", "q", "t"], ["out1", "s", "p", "t", "q", "out0"],
                ["s", "p", "t", "q"], ["p", "q", "out0", "s", "t"]][case]
    b_labels = [["t", "v", "s", "out2"], ["out2", "t", "v", "s"], ["t", "s", "out2", "v"],
                ["s", "out1", "out2", "t"]][case]
    A = _rand(rng, [dims[l] for l in a_labels], np.complex64)
    B = _rand(rng, [dims[l] for l in b_labels], np.complex64)
    late = tc.LateBits(torch.zeros((3, 64), dtype=torch.int32, device="cuda"),
                       {"out0": 0, "out1": 1, "out2": 2})
    prev = tc.set_gemm_mode(mode)
    try:
        got = tc.contract_late(tc.Tensor(a_labels, A), tc.Tensor(b_labels, B), late)
        want = tc.contract(tc.Tensor(a_labels, A), tc.Tensor(b_labels, B))
    finally:
        tc.set_gemm_mode(prev)
    assert sorted(got.labels) == sorted(want.labels)
    w = want.transpose_to(got.labels).array
    assert np.linalg.norm(got.array - w) / np.linalg.norm(w) < 1e-5
    outs = [l for l in got.labels if l.startswith("out")]
    assert list(got.labels[:len(outs)]) == outs   # open outputs lead


@pytest.mark.parametrize("mode", ["auto", "ffma", "tc3"])
@pytest.mark.parametrize("case", range(4))
def test_late_batched_times_open_site(mode, case):
    """A batched intermediate times a tensor whose outputs are still open:
    the small operand's slice per bit-string is read in place through B
    entry offsets (qf_cgemm_c64_ex b_boff) -- equals slicing it first."""
    rng = np.random.default_rng(500 + case)
    nb = [64, 17, 128, 1024][case]
    dims = {"p": 8, "q": 8, "s": 8, "t": 8, "v": 8, "out0": 2, "out1": 2}
    a_labels = [["@b", "p", "q", "s", "t"], ["@b", "s", "p", "t", "q"], ["@b", "t", "s", "p", "q"],
                ["@b", "p", "s", "q", "t"]][case]
    b_labels = [["t", "s", "v", "out0"], ["out1", "t", "v", "s", "out0"], ["s", "out0", "t"],
                ["t", "v", "s", "out1"]][case]
    outs = [l for l in b_labels if l.startswith("out")]
    A = _rand(rng, [nb] + [dims[l] for l in a_labels[1:]], np.complex64)
    Bm = _rand(rng, [dims[l] for l in b_labels], np.complex64)
    bits = rng.integers(0, 2, size=(2, nb)).astype(np.int32)
    late = tc.LateBits(torch.from_numpy(bits).cuda(), {"out0": 0, "out1": 1})
    prev = tc.set_gemm_mode(mode)
    try:
        ta, tb = tc.Tensor(a_labels, A), tc.Tensor(b_labels, Bm)
        got = tc.contract_late(ta, tb, late)
        want = tc.contract(ta, late.batch(tb))
    finally:
        tc.set_gemm_mode(prev)
    assert sorted(got.labels) == sorted(want.labels)
    w = want.transpose_to(got.labels).array
    assert np.linalg.norm(got.array - w) / np.linalg.norm(w) < 1e-5


@pytest.mark.parametrize("mode", ["auto", "ffma", "tc3"])
@pytest.mark.parametrize("nb", [8, 256])
def test_cut_slice_view_read_in_place(mode, nb):
    """Slice-late cuts: with the kept-open cut index right after the batch
    axis, a per-path fix is a strided view that the next late-sliced GEMM
    reads in place -- equal to fixing (copying) first."""
    rng = np.random.default_rng(600 + nb)
    A = _rand(rng, (nb, 4, 8, 8, 8), np.complex64)                 # @b c p q s
    W = _rand(rng, (8, 8, 2), np.complex64)                        # p q out1
    bits = rng.integers(0, 2, size=(2, nb)).astype(np.int32)
    late = tc.LateBits(torch.from_numpy(bits).cuda(), {"out0": 0, "out1": 1})
    prev = tc.set_gemm_mode(mode)
    try:
        lead = tc.Tensor(["@b", "c", "p", "q", "s"], A)
        tw = tc.Tensor(["p", "q", "out1"], W)
        for v in (0, 3):
            view = lead.fix_view("c", v)
            assert view._data is None
            got = tc.contract_late(view, tw, late)
            assert view._data is None                               # read in place
            want = tc.contract(lead.fix("c", v), late.batch(tw))
            w = want.transpose_to(got.labels).array
            assert np.linalg.norm(got.array - w) / np.linalg.norm(w) < 1e-5
            np.testing.assert_array_equal(view.array, lead.fix("c", v).array)
        mid = lead.fix_view("q", 1)                                 # not leading: plain fix
        assert mid._data is not None
    finally:
        tc.set_gemm_mode(prev)


@pytest.mark.parametrize("case", range(5))
def test_tma_view_of_scattered_operand(case):
    """Big operand whose innermost label is summed and whose other summed
    label sits between its free labels: read as a 5-D TMA view
    (qf_cgemm_c64_view) -- equal to the offset-table path and to numpy."""
    rng = np.random.default_rng(700 + case)
    nb = [4, 64, 1, 16, 32][case]
    dims = {"p": 8, "q": 16, "r": 8, "s": 8, "t": 8, "u": 4, "v": 8, "w": 8}
    a_labels = [["@b", "p", "s", "q", "r", "t"], ["@b", "s", "p", "q", "t"],
                ["@b", "q", "s", "p", "u", "t"], ["@b", "p", "q", "s", "t"],
                ["@b", "u", "s", "p", "r", "t"]][case]
    b_labels = ["@b", "s", "t", "v", "w"]
    A = _rand(rng, [nb] + [dims[l] for l in a_labels[1:]], np.complex64)
    B = _rand(rng, [nb] + [dims[l] for l in b_labels[1:]], np.complex64)
    outs = []
    for view in (True, False):
        prev = tc.set_view(view)
        try:
            with tc.KernelTimer() as kt:
                o = tc.contract(tc.Tensor(a_labels, A), tc.Tensor(b_labels, B))
            kinds = kt.summary(detail=True)
        finally:
            tc.set_view(prev)
        outs.append(o)
        if view and case != 3:   # case 3: s, t adjacent -> plain N layout, no view needed
            assert any(" V" in k for k in kinds), kinds
    keep = outs[0].labels
    ref_l = outs[1].transpose_to(keep).array
    assert np.linalg.norm(outs[0].array - ref_l) / np.linalg.norm(ref_l) < 1e-6
    sub = {l: chr(ord("a") + i) for i, l in enumerate(["@b"] + list(dims))}
    spec = "".join(sub[l] for l in a_labels) + "," + "".join(sub[l] for l in b_labels) + "->" + \
        "".join(sub[l] for l in keep)
    ref = np.einsum(spec, A.astype(np.complex128), B.astype(np.complex128))
    assert np.linalg.norm(outs[0].array - ref) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("nb", [8, 300])
def test_tma_view_with_sliced_site(nb):
    """Late slicing + view: batched big operand read as a TMA view, the site's
    per-bit-string slice as a TMA coordinate (b_boff / b_nslice)."""
    rng = np.random.default_rng(800 + nb)
    A = _rand(rng, (nb, 8, 8, 8, 8, 8), np.complex64)        # @b p s q r t
    S = _rand(rng, (8, 8, 8, 8, 2), np.complex64)            # s t v w out0
    bits = rng.integers(0, 2, size=(1, nb)).astype(np.int32)
    late = tc.LateBits(torch.from_numpy(bits).cuda(), {"out0": 0})
    ta = tc.Tensor(["@b", "p", "s", "q", "r", "t"], A)
    ts = tc.Tensor(["s", "t", "v", "w", "out0"], S)
    with tc.KernelTimer() as kt:
        got = tc.contract_late(ta, ts, late)
    assert any(" V" in k for k in kt.summary(detail=True))
    want = tc.contract(ta, late.batch(ts))
    w = want.transpose_to(got.labels).array
    assert np.linalg.norm(got.array - w) / np.linalg.norm(w) < 1e-5


@pytest.mark.parametrize("nb", [4, 128])
@pytest.mark.parametrize("perm", [0, 1])
def test_transposed_store_for_kept_cut(nb, perm):
    """Slice-late: a kept cut that is the small operand's only free index is
    stored in front of the rows (qf_cgemm_c64_ex with QF_C_TRANS, row-block /
    row-stream epilogues) -- same values as the row-major result."""
    rng = np.random.default_rng(900 + nb + perm)
    a_labels = ["@b", "p", "q", "s", "t"] if perm == 0 else ["@b", "s", "p", "t", "q"]
    A = _rand(rng, (nb, 8, 8, 8, 8), np.complex64)
    S = _rand(rng, (8, 8, 8, 2), np.complex64)                     # s t c out0
    bits = rng.integers(0, 2, size=(1, nb)).astype(np.int32)
    late = tc.LateBits(torch.from_numpy(bits).cuda(), {"out0": 0})
    ta, ts = tc.Tensor(a_labels, A), tc.Tensor(["s", "t", "c", "out0"], S)
    got = tc.contract_late(ta, ts, late, lead=("c",))
    assert got.labels[:2] == ("@b", "c")
    want = tc.contract(ta, late.batch(ts))
    w = want.transpose_to(got.labels).array
    assert np.linalg.norm(got.array - w) / np.linalg.norm(w) < 1e-5


@pytest.mark.parametrize("shape", [(3, 4096, 8, 64), (1, 32768, 8, 8), (5, 1000, 8, 64),
                                   (7, 333, 5, 24), (2, 100, 3, 7), (4, 64, 1, 1),
                                   (2, 4096, 8, 33), (1, 96, 7, 64), (300, 256, 8, 16)])
@pytest.mark.parametrize("ops", [(0, 0), (1, 1), (0, 1), (1, 0)])
@pytest.mark.parametrize("ab", [(1.0, 0.0), (0.5 - 1j, 0.25 + 0.5j)])
def test_rowmma_narrow_outputs(shape, ops, ab):
    """N <= 8, K <= 64: the row-stream pipeline on warp-level tensor cores
    (mma.sync TF32, 3xTF32) -- every layout, alpha/beta, ragged K and rows."""
    lib = _lib.load()
    prev = lib.qf_rowmma(1)
    try:
        assert _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_AUTO, alpha=ab[0], beta=ab[1]) < 1e-5
        gemv = shape[2] <= 4 and ops[0] == 0 and shape[3] >= 32   # warp-per-row GEMV first
        if shape[1] >= 32 and not gemv:
            assert lib.qf_last_kernel() == b"cgemm_rowmma"
        lib.qf_rowmma(0)
        assert _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_AUTO, alpha=ab[0], beta=ab[1]) < 1e-5
        lib.qf_rowmma(1)
        _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_FFMA)
        assert lib.qf_last_kernel() != b"cgemm_rowmma"      # the FFMA baseline stays FFMA
    finally:
        lib.qf_rowmma(prev)


@pytest.mark.parametrize("shape", [(1, 64, 1, 1 << 20), (2, 16, 4, 5000), (1, 200, 1, 777),
                                   (3, 8, 3, 4096), (1, 256, 1, 300)])
@pytest.mark.parametrize("ops", [(0, 0), (0, 1)])
def test_skinny_many_rows(shape, ops):
    """M*N <= 256 outputs, long K, row-contiguous A: warp-per-row split-K."""
    assert _gemm(*shape, *ops, np.complex64) < 1e-5
    assert _gemm(*shape, *ops, np.complex64, alpha=0.5 + 1j, beta=-0.25) < 1e-5


@pytest.mark.parametrize("shape", [(2, 8192, 8, 8, 64), (1, 4096, 3, 5, 32), (3, 2048, 16, 16, 256),
                                   (2, 96, 8, 64, 32), (1, 1000, 8, 8, 40)])
def test_rowblocks_gemm(shape):
    """A read in row blocks ([outer rows][k][inner rows], qf_cgemm_c64_rowblocks)."""
    import ctypes
    nb, M, N, K, rin = shape
    if M % rin:
        M = (M // rin + 1) * rin
    rng = np.random.default_rng(7)
    A = _rand(rng, (M // rin, K, rin), np.complex64)          # broadcast over the batch
    B = _rand(rng, (nb, K, N), np.complex64)
    dA, dB = torch.from_numpy(A.reshape(-1)).cuda(), torch.from_numpy(B.reshape(-1)).cuda()
    dC = torch.empty(nb * M * N, dtype=torch.complex64, device="cuda")
    lib = _lib.load()
    st = lib.qf_cgemm_c64_rowblocks(0, nb, M, N, K, ctypes.c_void_p(dA.data_ptr()), rin, rin * K,
                                    rin, 0, ctypes.c_void_p(dB.data_ptr()), N, K * N, 0,
                                    ctypes.c_void_p(dC.data_ptr()), N, M * N, 1.0, 0.0, 0.0, 0.0,
                                    tc.stream_handle())
    _lib.check(st, "rowblocks")
    a2 = A.transpose(0, 2, 1).reshape(M, K).astype(np.complex128)    # rows = (outer, inner)
    want = np.einsum("mk,bkn->bmn", a2, B.astype(np.complex128))
    got = dC.cpu().numpy().reshape(nb, M, N)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5


def test_open_step_with_too_many_rows_reads_row_blocks():
    """_contract_open beyond the offset-table limit: [outer][k][inner] big
    operand read in place (no permute) -- same result as the permuted path."""
    rng = np.random.default_rng(11)
    big = tc.Tensor(["o0", "a", "b", "c", "k", "d", "e"],
                    _rand(rng, (2, 64, 64, 16, 8, 8, 8), np.complex64))   # 2^23 rows x k 8
    small = tc.Tensor(["out1", "k", "n"], _rand(rng, (2, 8, 8), np.complex64))
    bits = torch.zeros((2, 4), dtype=torch.int32, device="cuda")
    late = tc.LateBits(bits, {"o0": 0, "out1": 1}, limit=2 ** 20)
    with tc.KernelTimer() as kt:
        got = tc._contract_open(big, small, late)
    kinds = kt.summary()
    assert "permute" not in kinds
    want = np.einsum("oabckde,pkn->poabcden", big.array, small.array)
    w = np.moveaxis(want, 0, 0)   # labels: out1, o0, a, b, c, d, e, n
    assert got.labels == ("out1", "o0", "a", "b", "c", "d", "e", "n")
    g = got.array
    assert np.linalg.norm(g - w) / np.linalg.norm(w) < 1e-5


@pytest.mark.parametrize("shape", [(1024, 1, 1, 4096), (700, 1, 1, 64), (600, 1, 1, 1000),
                                   (2048, 1, 1, 130), (600, 1, 1, 999)])
@pytest.mark.parametrize("ops", [(0, 0), (0, 1)])
@pytest.mark.parametrize("ab", [(1.0, 0.0), (0.5 - 1j, 0.25 + 0.5j)])
def test_batched_dot_products(shape, ops, ab):
    """M = N = 1 with many entries: the warp-per-entry dot kernel (odd K and
    short K fall back to the split-K kernel) against float64."""
    assert _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_FFMA, alpha=ab[0], beta=ab[1]) < 1e-5
    assert _gemm(*shape, *ops, np.complex64, alpha=ab[0], beta=ab[1]) < 1e-5


@pytest.mark.parametrize("case", range(6))
@pytest.mark.parametrize("kept", [False, True])
def test_transposed_tma_view(case, kept):
    """Big operand whose innermost labels are FREE rows, summed labels in one
    or two runs around them ([ko][rb][ki][ra] and friends): read as a
    transposed 5-D TMA view (qf_cgemm_c64_tview; non-monotonic map strides),
    with a per-bit-string site slice and, for a kept cut, the transposed
    tensor-core epilogue -- equal to the engines without the view and to
    float64 numpy."""
    rng = np.random.default_rng(1100 + case + 10 * kept)
    nb = [8, 64, 3, 16, 32, 5][case]
    dims = {"p": 8, "q": 8, "r": 8, "s": 8, "t": 8, "u": 16, "x": 2}
    a_labels = [["@b", "s", "p", "q", "r", "t", "u"],      # [ko][rb][ki][ra]
                ["@b", "s", "p", "q", "t", "r"],           # [ko][rb][ki][ra]
                ["@b", "p", "q", "s", "t", "r"],           # [rb][k][ra]
                ["@b", "s", "t", "p", "q", "r"],           # [k][ra] (one row run)
                ["@b", "p", "s", "q", "t", "r", "u"],      # [rb][ko][rb'] -> 3 free runs: no view
                ["@b", "s", "p", "t", "x", "q"]][case]     # ra = 16 rows (x, q)
    ks = ["s", "t"]
    A = _rand(rng, [nb] + [dims[l] for l in a_labels[1:]], np.complex64)
    S = _rand(rng, (8, 8, 8, 2), np.complex64)                     # s t c out0
    bits = rng.integers(0, 2, size=(1, nb)).astype(np.int32)
    late = tc.LateBits(torch.from_numpy(bits).cuda(), {"out0": 0})
    ta, ts = tc.Tensor(a_labels, A), tc.Tensor(["s", "t", "c", "out0"], S)
    lead = ("c",) if kept else ()
    outs = []
    for tv in (True, False):
        prev = tc.set_tview(tv)
        try:
            with tc.KernelTimer() as kt:
                o = tc.contract_late(ta, ts, late, lead=lead)
            kinds = kt.summary(detail=True)
        finally:
            tc.set_tview(prev)
        outs.append(o)
        if tv and case not in (3, 4):   # 3: plain opA = T layout; 4: three free runs
            assert any(" TV" in k for k in kinds), kinds
    if kept:
        assert outs[0].labels[:2] == ("@b", "c")
    ref_t = outs[1].transpose_to(outs[0].labels).array
    assert np.linalg.norm(outs[0].array - ref_t) / np.linalg.norm(ref_t) < 1e-5
    want = tc.contract(ta, late.batch(ts))
    w = want.transpose_to(outs[0].labels).array
    assert np.linalg.norm(outs[0].array - w) / np.linalg.norm(w) < 1e-5
    assert [l for l in a_labels if l in ks]   # summed labels present


@pytest.mark.parametrize("nb", [4, 130])
@pytest.mark.parametrize("ra", [8, 16])
def test_reassociated_expansion_matches_two_contractions(nb, ra):
    """(T . S) . W run as T . (S . W) (expand_plan / contract_late_expand: one
    batched GEMM per bit-string with its block of S . W picked by TMA slice
    coordinate; the wide T . S intermediate is never written) -- equal to
    the two late-sliced contractions and to float64 numpy."""
    rng = np.random.default_rng(1300 + nb + ra)
    T = _rand(rng, (nb, 8, 16, 8, 8), np.complex64)              # @b p q r(ko) s(j)
    S = _rand(rng, (8, ra, 8, 2), np.complex64)                  # s(j) t(ra) u(ki) out0
    W = _rand(rng, (8, 8, 4, 16, 2), np.complex64)               # r(ko) u(ki) v w out1
    bits = rng.integers(0, 2, size=(2, nb)).astype(np.int32)
    late = tc.LateBits(torch.from_numpy(bits).cuda(), {"out0": 0, "out1": 1})
    tt = tc.Tensor(["@b", "p", "q", "r", "s"], T)
    ts = tc.Tensor(["s", "t", "u", "out0"], S)
    tw = tc.Tensor(["r", "u", "v", "w", "out1"], W)
    plan = tc.expand_plan(tt, ts, tw, late)
    assert plan is not None
    with tc.KernelTimer() as kt:
        got = tc.contract_late_expand(tt, ts, tw, late, plan)
    assert got is not None and any(" X" in k for k in kt.summary(detail=True))
    u = tc.contract_late(tt, ts, late, tail=("r", "u", "v", "w", "out1"))
    want = tc.contract_late(u, tw, late)
    assert got.labels == want.labels
    w = want.array
    assert np.linalg.norm(got.array - w) / np.linalg.norm(w) < 1e-5
    sb = np.take_along_axis(S[None].repeat(nb, 0), bits[0][:, None, None, None, None], 4)[..., 0]
    wb = np.take_along_axis(W[None].repeat(nb, 0), bits[1][:, None, None, None, None, None], 5)[..., 0]
    ref = np.einsum("bpqrs,bstu,bruvw->bpqtvw", T.astype(np.complex128), sb.astype(np.complex128),
                    wb.astype(np.complex128))
    g = got.transpose_to(("@b", "p", "q", "t", "v", "w")).array
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("nb", [8, 200])
@pytest.mark.parametrize("ra", [1, 4])
def test_reassociated_expansion_open_operand(nb, ra):
    """expand_plan with acc still carrying open outputs: each bit-string's
    slice of acc read in place as a TMA view at a slice coordinate
    (qf_cgemm_c64_view2 a_boff / a_nslice), times its block of S . W --
    equal to the two late contractions and to float64 numpy."""
    rng = np.random.default_rng(1400 + nb + ra)
    A = _rand(rng, (2, 2, 8, 16, 8, 8, 8), np.complex64)        # o0 o1 p q j r ko
    s_lab = ["j", "u", "out2"] if ra == 1 else ["j", "t", "u", "out2"]
    S = _rand(rng, (8, 8, 2) if ra == 1 else (8, ra, 8, 2), np.complex64)
    W = _rand(rng, (8, 8, 8, 2), np.complex64)                  # ko u w out3
    bits = rng.integers(0, 2, size=(4, nb)).astype(np.int32)
    late = tc.LateBits(torch.from_numpy(bits).cuda(), {"o0": 0, "o1": 1, "out2": 2, "out3": 3},
                       limit=8)
    ta = tc.Tensor(["o0", "o1", "p", "q", "j", "r", "ko"], A)
    ts, tw = tc.Tensor(s_lab, S), tc.Tensor(["ko", "u", "w", "out3"], W)
    plan = tc.expand_plan(ta, ts, tw, late)
    assert plan is not None and plan.get("open")
    with tc.KernelTimer() as kt:
        got = tc.contract_late_expand(ta, ts, tw, late, plan)
    assert got is not None and any(" XO" in k or " XK" in k for k in kt.summary(detail=True))
    if plan.get("keep_open"):           # outputs kept open: slice the bit-strings out
        got = late.batch(got)
    u = tc.contract_late(ta, ts, late, tail=("ko", "u", "w", "out3"))
    want = tc.contract_late(u, tw, late)
    w = want.transpose_to(got.labels).array
    assert np.linalg.norm(got.array - w) / np.linalg.norm(w) < 1e-5
    o = bits.T
    ab = A[o[:, 0], o[:, 1]]                                      # b p q j r ko
    sb = S[..., o[:, 2]]
    sb = np.moveaxis(sb, -1, 0)
    wb = np.moveaxis(W[..., o[:, 3]], -1, 0)
    if ra == 1:
        ref = np.einsum("bpqjrk,bju,bkuw->bpqrw", ab.astype(np.complex128),
                        sb.astype(np.complex128), wb.astype(np.complex128))
        g = got.transpose_to(("@b", "p", "q", "r", "w")).array
    else:
        ref = np.einsum("bpqjrk,bjtu,bkuw->bpqrtw", ab.astype(np.complex128),
                        sb.astype(np.complex128), wb.astype(np.complex128))
        g = got.transpose_to(("@b", "p", "q", "r", "t", "w")).array
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("nb", [4, 64])
@pytest.mark.parametrize("wide", [False, True])
def test_reassociated_expansion_view_operand(nb, wide):
    """expand_plan on a batched operand whose summed labels straddle its rows
    ([@b][ko][p][q][j...]): acc read as a TMA view (qf_cgemm_c64_view2; K up
    to 512 through the promoted long-K kernel) times its block of S . W."""
    rng = np.random.default_rng(1500 + nb + wide)
    jd = (8, 8) if wide else (8,)
    A = _rand(rng, (nb, 8, 8, 16) + jd, np.complex64)           # @b r(ko) p q j..
    j_lab = ["j1", "j2"] if wide else ["j1"]
    S = _rand(rng, jd + (8, 8, 2), np.complex64)                # j.. t(ra) u(ki) out0
    W = _rand(rng, (8, 8, 8, 2), np.complex64)                  # r(ko) u(ki) v out1
    bits = rng.integers(0, 2, size=(2, nb)).astype(np.int32)
    late = tc.LateBits(torch.from_numpy(bits).cuda(), {"out0": 0, "out1": 1})
    ta = tc.Tensor(["@b", "r", "p", "q"] + j_lab, A)
    ts = tc.Tensor(j_lab + ["t", "u", "out0"], S)
    tw = tc.Tensor(["r", "u", "v", "out1"], W)
    plan = tc.expand_plan(ta, ts, tw, late)
    assert plan is not None and plan["view"] is not None
    with tc.KernelTimer() as kt:
        got = tc.contract_late_expand(ta, ts, tw, late, plan)
    assert got is not None and any(" XV" in k for k in kt.summary(detail=True))
    u = tc.contract_late(ta, ts, late, tail=("r", "u", "v", "out1"))
    want = tc.contract_late(u, tw, late)
    w = want.transpose_to(got.labels).array
    assert np.linalg.norm(got.array - w) / np.linalg.norm(w) < 1e-5


@pytest.mark.parametrize("nb", [64, 300])
def test_reassociated_expansion_keeps_outputs_open(nb):
    """expand_plan on an open operand when every (slice, output) combination
    is at most the bit-string count: all combinations in one pass with the
    outputs kept open (column-blocked C through qf_cgemm_c64_view2), then the
    next re-associated pair reads its per-bit-string slices by TMA slice
    coordinate (qf_cgemm_c64_ex2 a_nslice) -- equal to the plain late walk."""
    rng = np.random.default_rng(1600 + nb)
    A = _rand(rng, (2, 2, 8, 16, 8, 8, 8), np.complex64)        # o0 o1 p q j r ko
    S = _rand(rng, (8, 8, 2), np.complex64)                     # j u out2
    W = _rand(rng, (8, 8, 8, 2), np.complex64)                  # ko u w out3
    S2 = _rand(rng, (8, 4, 8, 2), np.complex64)                 # w x y out4
    W2 = _rand(rng, (8, 8, 8, 2), np.complex64)                 # r y z out5
    bits = rng.integers(0, 2, size=(6, nb)).astype(np.int32)
    late = tc.LateBits(torch.from_numpy(bits).cuda(),
                       {"o0": 0, "o1": 1, "out2": 2, "out3": 3, "out4": 4, "out5": 5}, limit=8)
    ta = tc.Tensor(["o0", "o1", "p", "q", "j", "r", "ko"], A)
    ts, tw = tc.Tensor(["j", "u", "out2"], S), tc.Tensor(["ko", "u", "w", "out3"], W)
    ts2, tw2 = tc.Tensor(["w", "x", "y", "out4"], S2), tc.Tensor(["r", "y", "z", "out5"], W2)
    plan = tc.expand_plan(ta, ts, tw, late)
    assert plan is not None and plan.get("keep_open")
    with tc.KernelTimer() as kt:
        t_open = tc.contract_late_expand(ta, ts, tw, late, plan)
        plan2 = tc.expand_plan(t_open, ts2, tw2, late)
        assert plan2 is not None and plan2.get("sliced")
        got = tc.contract_late_expand(t_open, ts2, tw2, late, plan2)
    kinds = kt.summary(detail=True)
    assert any(" XK" in k for k in kinds) and got is not None, kinds
    u = tc.contract_late(ta, ts, late, tail=("ko", "u", "w", "out3"))
    t = tc.contract_late(u, tw, late)
    u2 = tc.contract_late(t, ts2, late, tail=("r", "y", "z", "out5"))
    want = tc.contract_late(u2, tw2, late)
    w = want.transpose_to(got.labels).array
    assert np.linalg.norm(got.array - w) / np.linalg.norm(w) < 1e-5


# ---------------------------------------------------------------------------
# library-owned state vs CUDA graphs


def test_skinny_batch_beyond_grid_limit_c128():
    """The split-K skinny path (M*N <= 256, K >= 256) carries the batch in
    gridDim.y; more than 65535 entries are split into several launches."""
    assert _gemm(70000, 1, 1, 256, 0, 1, np.complex128) < 1e-12


def test_graph_replay_survives_workspace_growth():
    """A captured split-K GEMM keeps the workspace pointer it saw: a later,
    larger eager GEMM must not free it under the graph."""
    rng = np.random.default_rng(11)
    b, K = 64, 4096
    A = torch.from_numpy(_rand(rng, (b, 1, K), np.complex64).reshape(-1)).cuda()
    B = torch.from_numpy(_rand(rng, (b, K, 1), np.complex64).reshape(-1)).cuda()
    C = torch.zeros(b, dtype=torch.complex64, device="cuda")
    run = lambda: tc.gemm_buffer(b, 1, 1, K, A, 0, B, 0, C, mode=_lib.GEMM_FFMA)  # noqa: E731
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        run()                                  # warm-up reserves the workspace
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        run()
    want = C.clone()
    # a larger split-K call (16 x 16 outputs per entry: > 1 MiB of partials)
    # grows the workspace eagerly
    b2, M2, K2 = 500, 16, 8192
    A2 = torch.randn(b2 * M2 * K2, dtype=torch.complex64, device="cuda")
    B2 = torch.randn(b2 * K2 * M2, dtype=torch.complex64, device="cuda")
    C2 = torch.empty(b2 * M2 * M2, dtype=torch.complex64, device="cuda")
    tc.gemm_buffer(b2, M2, M2, K2, A2, 0, B2, 0, C2, mode=_lib.GEMM_FFMA)
    del A2, B2
    C.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(C, want)


def test_permute_plan_first_built_in_capture_is_refused():
    x = torch.randn(2 ** 12, dtype=torch.complex64, device="cuda")
    y = torch.empty_like(x)
    dims, perm = [2] * 12, [11, 3, 7, 0, 10, 1, 9, 2, 8, 4, 6, 5]
    g = torch.cuda.CUDAGraph()
    with pytest.raises(Exception):
        with torch.cuda.graph(g):
            tc.permute_buffer(x, dims, perm, out=y)
    torch.cuda.synchronize()
    tc.permute_buffer(x, dims, perm, out=y)          # eager: plan built
    g2 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2):                        # now capturable (and pinned)
        tc.permute_buffer(x, dims, perm, out=y)
    y.zero_()
    g2.replay()
    torch.cuda.synchronize()
    want = x.cpu().numpy().reshape(dims).transpose(perm).reshape(-1)
    assert np.array_equal(y.cpu().numpy(), want)


# wide (128 x 128 tile) Gauss long-K kernel, qf_gemm_tcw.cu: full and ragged
# tiles in M, N and K, several tiles per CTA, entries (batch), all operand
# layouts, 1/2/many promotion chunks per tile
WIDE_SHAPES = [(1, 256, 256, 1024), (1, 128, 128, 512), (2, 384, 640, 520), (1, 1000, 1152, 778),
               (3, 2048, 1024, 1024), (1, 19000, 128, 512), (1, 128, 2048, 4100),
               # K >= 2048: the TMA producers run in lockstep epochs; more tiles than
               # CTAs / CTA pairs with a ragged last wave (CTAs with fewer tiles
               # pre-arrive for the epochs they never reach), several entries
               (1, 19200, 128, 2048), (2, 9500, 256, 2056)]


@pytest.mark.parametrize("shape", WIDE_SHAPES)
@pytest.mark.parametrize("ops", [(0, 0), (1, 1), (0, 1), (1, 0)])
@pytest.mark.parametrize("variant", [40, 41, 42, 43, 44, 46],
                         ids=["ck64", "ck128", "ck32", "pair-ck64", "pair-ck128", "pair-drain4"])
def test_tcgen05_wide_gauss_long_k(shape, ops, variant):
    lib = _lib.load()
    prev = lib.qf_tc3_set_variant(variant)
    try:
        err = _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_TC3)
        assert _lib.last_kernel() == "cgemm_tc3w"
    finally:
        lib.qf_tc3_set_variant(prev)
    assert err < 1e-5, err


@pytest.mark.parametrize("K", [4096, 32768])
@pytest.mark.parametrize("variant", [40, 41, 43], ids=["ck64", "ck128", "pair-ck64"])
def test_tcgen05_wide_accuracy_at_long_k(K, variant):
    lib = _lib.load()
    prev = lib.qf_tc3_set_variant(variant)
    try:
        err = _gemm(1, 256, 256, K, 0, 0, np.complex64, mode=_lib.GEMM_TC3)
    finally:
        lib.qf_tc3_set_variant(prev)
    assert err < (1e-5 if variant == 41 else 5e-6), err


@pytest.mark.parametrize("ab", [(0.5 - 1j, 0.0), (1.0, 0.5 + 0.25j)])
@pytest.mark.parametrize("variant", [40, 43], ids=["single", "pair"])
def test_tcgen05_wide_alpha_beta(ab, variant):
    lib = _lib.load()
    prev = lib.qf_tc3_set_variant(variant)
    try:
        err = _gemm(2, 300, 384, 1024, 0, 1, np.complex64, _lib.GEMM_TC3, ab[0], ab[1])
    finally:
        lib.qf_tc3_set_variant(prev)
    assert err < 1e-5, err


@pytest.mark.parametrize("case", range(3))
def test_long_k_view_on_the_wide_kernel(case):
    """A compute-bound contraction whose big operand has its summed labels in
    two runs: read in place as a 5-D TMA view by the wide long-K kernel
    (single CTAs and CTA pairs) instead of being permuted first -- equal to
    the permuted path and to numpy."""
    rng = np.random.default_rng(900 + case)
    dims = {"r0": [16, 8, 40][case], "k0": 16, "r1": [256, 128, 64][case], "k1": [16, 32, 16][case],
            "n": [256, 128, 384][case]}
    a_labels, b_labels = ["r0", "k0", "r1", "k1"], ["k0", "k1", "n"]
    A = _rand(rng, [dims[l] for l in a_labels], np.complex64)
    B = _rand(rng, [dims[l] for l in b_labels], np.complex64)
    ref = np.einsum("akbl,kln->abn", A.astype(np.complex128), B.astype(np.complex128))
    lib = _lib.load()
    for variant in (0, 40, 43):
        prev = lib.qf_tc3_set_variant(variant)
        try:
            with tc.KernelTimer() as kt:
                o = tc.contract(tc.Tensor(a_labels, A), tc.Tensor(b_labels, B))
            kinds = kt.summary(detail=True)
        finally:
            lib.qf_tc3_set_variant(prev)
        assert any(" V" in k for k in kinds), kinds
        assert _lib.last_kernel() == "cgemm_tc3w"
        assert o.labels == ("r0", "r1", "n")
        assert np.linalg.norm(o.array - ref) / np.linalg.norm(ref) < 1e-5
    prev = tc.set_view(False)
    try:
        o2 = tc.contract(tc.Tensor(a_labels, A), tc.Tensor(b_labels, B))
    finally:
        tc.set_view(prev)
    assert np.linalg.norm(o2.array - ref) / np.linalg.norm(ref) < 1e-5


@pytest.mark.parametrize("variant", [32, 40, 43], ids=["narrow", "wide", "wide-pair"])
@pytest.mark.parametrize("ops", [(0, 0), (0, 1)])
def test_long_k_slice_coordinates(variant, ops):
    """qf_cgemm_c64_ex2 at a long-K shape: every entry picks its A entry and
    its [K][N] B slice by offset (a_boff / a_nslice, b_boff / b_nslice), which
    the TMA-fed long-K kernels (64-column and wide, single CTAs and pairs)
    turn into slice coordinates."""
    import ctypes
    rng = np.random.default_rng(77)
    nb, M, N, K, a_ns, b_ns = 6, 256, 128, 512, 4, 3
    opA, opB = ops
    A = _rand(rng, (a_ns, M, K), np.complex64)
    B = _rand(rng, (b_ns, K, N) if opB == 0 else (b_ns, N, K), np.complex64)
    pa, pb = rng.integers(0, a_ns, size=nb), rng.integers(0, b_ns, size=nb)
    dA, dB = torch.from_numpy(A.reshape(-1)).cuda(), torch.from_numpy(B.reshape(-1)).cuda()
    a_boff = torch.from_numpy((pa * M * K).astype(np.int64)).cuda()
    b_boff = torch.from_numpy((pb * K * N).astype(np.int64)).cuda()
    out = torch.zeros(nb * M * N, dtype=torch.complex64, device="cuda")
    lib = _lib.load()
    vp = ctypes.c_void_p
    prev = lib.qf_tc3_set_variant(variant)
    try:
        st = lib.qf_cgemm_c64_ex2(
            _lib.GEMM_TC3 | _lib.BOFF_EVEN | _lib.BBOFF_EVEN, nb, M, N, K, vp(dA.data_ptr()), K, M * K,
            _lib.OP_N, vp(a_boff.data_ptr()), a_ns, vp(0), vp(0), vp(dB.data_ptr()),
            N if opB == 0 else K, K * N, opB, vp(b_boff.data_ptr()), b_ns, vp(out.data_ptr()), N,
            M * N, 1.0, 0.0, 0.0, 0.0, tc.stream_handle())
        _lib.check(st, "ex2")
        torch.cuda.synchronize()
        kern = _lib.last_kernel()
    finally:
        lib.qf_tc3_set_variant(prev)
    assert kern == ("cgemm_tc3g" if variant == 32 else "cgemm_tc3w"), kern
    Bn = B if opB == 0 else B.transpose(0, 2, 1)
    want = np.matmul(A[pa].astype(np.complex128), Bn[pb].astype(np.complex128))
    got = out.cpu().numpy().reshape(nb, M, N)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5


# streaming kernel (qf_gemm_tcs.cu): one entry, huge M, K = 16, N = 16 / 32;
# ragged last tile, both B layouts, alpha, more tiles than CTAs
@pytest.mark.parametrize("shape", [(1, 128 * 148, 16, 16), (1, 40000, 16, 16), (1, 128 * 148 + 77, 32, 16),
                                   (1, 131072, 32, 16)])
@pytest.mark.parametrize("ops", [(0, 0), (0, 1)])
@pytest.mark.parametrize("alpha", [1.0, 0.5 - 1j])
def test_tcgen05_streaming_k16(shape, ops, alpha):
    err = _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_TC3, alpha=alpha)
    assert _lib.last_kernel() == "cgemm_tc3s"
    assert err < 1e-5, err
    # the generic short-K kernel on the same shape (pin 50) agrees
    lib = _lib.load()
    prev = lib.qf_tc3_set_variant(50)
    try:
        err2 = _gemm(*shape, *ops, np.complex64, mode=_lib.GEMM_TC3, alpha=alpha)
        assert _lib.last_kernel() != "cgemm_tc3s"
    finally:
        lib.qf_tc3_set_variant(prev)
    assert err2 < 1e-5, err2


@pytest.mark.parametrize("case", range(3))
def test_long_k_transposed_view_on_the_wide_kernel(case):
    """Compute-bound contraction whose big operand has its innermost labels
    FREE and its summed labels in two runs: read in place as a transposed 5-D
    TMA view by the wide long-K kernel (no permute) -- equal to numpy and to
    the permuted path."""
    rng = np.random.default_rng(950 + case)
    dims = {"k0": 16, "r0": [8, 4, 24][case], "k1": [16, 32, 16][case], "r1": [256, 128, 64][case],
            "n": [256, 128, 384][case]}
    a_labels, b_labels = ["k0", "r0", "k1", "r1"], ["k0", "k1", "n"]
    A = _rand(rng, [dims[l] for l in a_labels], np.complex64)
    B = _rand(rng, [dims[l] for l in b_labels], np.complex64)
    ref = np.einsum("kalb,kln->abn", A.astype(np.complex128), B.astype(np.complex128))
    lib = _lib.load()
    for variant in (0, 40, 43):
        prev = lib.qf_tc3_set_variant(variant)
        try:
            with tc.KernelTimer() as kt:
                o = tc.contract(tc.Tensor(a_labels, A), tc.Tensor(b_labels, B))
            kinds = kt.summary(detail=True)
        finally:
            lib.qf_tc3_set_variant(prev)
        assert any(" TV" in k for k in kinds), kinds
        assert _lib.last_kernel() == "cgemm_tc3w"
        assert o.labels == ("r0", "r1", "n")
        assert np.linalg.norm(o.array - ref) / np.linalg.norm(ref) < 1e-5
    prev = tc.set_tview(False)
    try:
        o2 = tc.contract(tc.Tensor(a_labels, A), tc.Tensor(b_labels, B))
    finally:
        tc.set_tview(prev)
    assert np.linalg.norm(o2.array - ref) / np.linalg.norm(ref) < 1e-5


def test_wide_kernel_with_lockstep_replays_from_a_cuda_graph():
    """A long-K GEMM on the wide kernel (lockstep counters zeroed by a memset
    node before the launch) captured in a CUDA graph: replays equal the eager
    result, also after other launches used the counter ring in between."""
    rng = np.random.default_rng(5)
    M, N, K = 4096, 256, 4096
    A = torch.from_numpy(_rand(rng, (M * K,), np.complex64)).cuda()
    B = torch.from_numpy(_rand(rng, (K * N,), np.complex64)).cuda()
    want = torch.empty(M * N, dtype=torch.complex64, device="cuda")
    tc.gemm_buffer(1, M, N, K, A, 0, B, 0, want, mode=_lib.GEMM_TC3)   # eager: allocates the ring
    assert _lib.last_kernel() == "cgemm_tc3w"
    out = torch.zeros_like(want)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        tc.gemm_buffer(1, M, N, K, A, 0, B, 0, out, mode=_lib.GEMM_TC3)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        tc.gemm_buffer(1, M, N, K, A, 0, B, 0, out, mode=_lib.GEMM_TC3)
    for _ in range(3):
        out.zero_()
        graph.replay()
        tc.gemm_buffer(1, M, N, K, A, 0, B, 0, want, mode=_lib.GEMM_TC3)   # rotates the ring
        torch.cuda.synchronize()
        assert torch.equal(out, want)


@pytest.mark.parametrize("case", [(1, 1000, 1152, 778, 40), (1, 1000, 1152, 778, 43), (2, 300, 384, 1024, 43),
                                  (1, 128 * 148 + 77, 16, 16, 0), (1, 40000, 32, 16, 0)],
                         ids=["wide-ragged", "pair-ragged", "pair-batch", "stream-n16", "stream-n32"])
def test_new_kernels_write_nothing_outside_c(case):
    """Canaries around C: ragged tiles of the wide kernel (register epilogue)
    and of the streaming kernel (TMA stores clip at M) leave every byte
    outside [C, C + batch*M*N) untouched."""
    b, M, N, K, variant = case
    rng = np.random.default_rng(31)
    A = torch.from_numpy(_rand(rng, (b * M * K,), np.complex64)).cuda()
    B = torch.from_numpy(_rand(rng, (b * K * N,), np.complex64)).cuda()
    pad = 4096
    big = torch.full((b * M * N + 2 * pad,), 7.0 - 3.0j, dtype=torch.complex64, device="cuda")
    C = big[pad:pad + b * M * N]
    lib = _lib.load()
    prev = lib.qf_tc3_set_variant(variant)
    try:
        tc.gemm_buffer(b, M, N, K, A, 0, B, 0, C, mode=_lib.GEMM_TC3)
        torch.cuda.synchronize()
        kern = _lib.last_kernel()
    finally:
        lib.qf_tc3_set_variant(prev)
    assert kern == ("cgemm_tc3s" if K == 16 else "cgemm_tc3w"), kern
    sentinel = torch.tensor(7.0 - 3.0j, dtype=torch.complex64, device="cuda")
    assert bool((big[:pad] == sentinel).all()) and bool((big[pad + b * M * N:] == sentinel).all())
    want = np.matmul(A.cpu().numpy().reshape(b, M, K).astype(np.complex128),
                     B.cpu().numpy().reshape(b, K, N).astype(np.complex128))
    got = C.cpu().numpy().reshape(b, M, N)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-5
