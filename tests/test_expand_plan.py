"""Host-side planning of the re-associated contractions (no GPU): which
(acc . op) . op2 triples run as acc . (op . op2), and how the big operand
is described (plain, TMA view, open slices).  Stand-in tensors carry only
the labels, dims and dtype that tensor_core.expand_plan reads."""

from __future__ import annotations

import math

import numpy as np
import torch

from paper_1811_09599_b200 import tensor_core as tc


class _Buf:
    dtype = torch.complex64


class FakeTensor:
    """labels/dims/dtype of a device tensor, nothing else."""

    def __init__(self, labels, dims):
        self.labels, self.dims = tuple(labels), tuple(dims)
        self.buf, self._data = _Buf(), object()

    @property
    def size(self):
        return math.prod(self.dims)


def _late(outs, nb, limit=None):
    bits = torch.zeros((len(outs), nb), dtype=torch.int32)
    return tc.LateBits(bits, {o: i for i, o in enumerate(outs)}, limit=limit)


def test_a_view_multi_label_runs():
    # [ko1 ko2][rows][ki]: the outer summed run of two adjacent labels is one axis
    labels = ["a", "b", "r1", "r2", "k"]
    dims = [8, 8, 16, 8, 8]
    v = tc._a_view(labels, dims, ["r1", "r2"], ["a", "b", "k"])
    assert v == (8, 128, 8, 64, 128 * 8, 1, 8 * 8 * 16 * 8 * 8)
    # three summed runs are not a view; neither is a non-memory-order k list
    assert tc._a_view(["a", "r", "b", "s", "k"], [8] * 5, ["r", "s"], ["a", "b", "k"]) is None
    assert tc._a_view(labels, dims, ["r1", "r2"], ["b", "a", "k"]) is None


def test_batched_widening_pair_is_reassociated():
    """config 2's 1024 x [512 rows][ko 8][j 8] . S(j, ra, ki, out) . W(ko, ki, w, out'):
    one 512 x 64 x 512 GEMM per bit-string instead of 4096x8x64 + 4096x64x64."""
    nb = 1024
    late = _late(["o1", "o2"], nb)
    acc = FakeTensor(["@b", "p", "q", "r", "ko", "j"], [nb, 8, 8, 8, 8, 8])
    op = FakeTensor(["ki", "j", "ra", "o1"], [8, 8, 8, 2])
    op2 = FakeTensor(["w1", "ko", "w2", "ki", "o2"], [8, 8, 8, 8, 2])
    plan = tc.expand_plan(acc, op, op2, late)
    assert plan is not None and plan["view"] is None and not plan["sliced"]
    assert (plan["M"], plan["K"], plan["N"]) == (512, 64, 512)
    assert plan["labels"] == ("@b", "p", "q", "r", "ra", "w1", "w2")
    # booked intermediate: the reference's acc . op
    assert set(plan["u"].labels) == {"@b", "p", "q", "r", "ko", "ra", "ki"}


def test_view_operand_and_flop_guard():
    nb = 1024
    late = _late(["o1", "o2"], nb)
    # ko outermost, j innermost: a TMA view with K = ko x j
    acc = FakeTensor(["@b", "ko", "p", "q", "r", "j1", "j2"], [nb, 8, 8, 8, 8, 8, 8])
    op = FakeTensor(["j1", "j2", "ki", "ra", "o1"], [8, 8, 8, 8, 2])
    op2 = FakeTensor(["ko", "ki", "cut", "o2"], [8, 8, 8, 2])
    plan = tc.expand_plan(acc, op, op2, late)
    assert plan is not None and plan["view"] is not None
    assert (plan["M"], plan["K"], plan["N"]) == (512, 512, 64)
    # a wide op2 would make the re-associated product dearer: refused
    wide = FakeTensor(["ko", "ki", "v", "w", "o2"], [8, 8, 8, 64, 2])
    assert tc.expand_plan(acc, op, wide, late) is None


def test_open_operand_kept_open_when_combinations_are_few():
    """acc with 8 open outputs (256 slices) . S(out) . W(out'): the reference
    slices at the second contraction (2^10 > limit 512); 256 x 4 combinations
    <= 1024 bit-strings, so all are computed once with outputs kept open."""
    nb = 1024
    outs = [f"o{i}" for i in range(8)] + ["s1", "s2"]
    late = _late(outs, nb)
    acc = FakeTensor(outs[:8] + ["a", "b", "c", "j", "r", "ko"], [2] * 8 + [8] * 6)
    op = FakeTensor(["j", "ki", "s1"], [8, 8, 2])
    op2 = FakeTensor(["ko", "ki", "w", "s2"], [8, 8, 8, 2])
    plan = tc.expand_plan(acc, op, op2, late)
    assert plan is not None and plan.get("open") and plan.get("keep_open")
    assert plan["labels"][:10] == tuple(outs)          # outputs lead the result
    # with fewer bit-strings than combinations: per-bit-string slices instead
    late_small = _late(outs, 128, limit=512)
    plan2 = tc.expand_plan(acc, op, op2, late_small)
    assert plan2 is None or not plan2.get("keep_open")


def test_sliced_open_operand_as_entries():
    """An open operand whose outputs exceed the limit: its per-bit-string
    slices are the GEMM entries (TMA slice coordinates)."""
    nb = 1024
    outs = [f"o{i}" for i in range(10)] + ["s1", "s2"]
    late = _late(outs, nb)
    acc = FakeTensor(outs[:10] + ["p", "q", "r", "ko", "j"], [2] * 10 + [8] * 5)
    op = FakeTensor(["ki", "j", "ra", "s1"], [8, 8, 8, 2])
    op2 = FakeTensor(["w1", "ko", "w2", "ki", "s2"], [8, 8, 8, 8, 2])
    plan = tc.expand_plan(acc, op, op2, late)
    assert plan is not None and plan["sliced"] and plan["nb"] == nb
    assert plan["labels"][0] == "@b"


def test_views_of_the_full_depth_region_builds():
    """The layouts the config-4/5 region builds meet (bond 32 / 16): summed
    labels in two runs.  Innermost summed -> row-major TMA view; innermost
    free -> transposed view; three free runs -> neither (permute)."""
    # config 5: [a0 .. a6] of 16, K = (a3, a6): rows (a0 a1 a2) x (a4 a5)
    labels, dims = [f"a{i}" for i in range(7)], [16] * 7
    kin, ra, sra, ko, sko, rb, srb = tc._a_view(labels, dims, ["a0", "a1", "a2", "a4", "a5"],
                                                ["a3", "a6"])
    assert (kin, ko, ra, rb) == (16, 16, 256, 4096)
    assert (sra, sko, srb) == (16, 16 ** 3, 16 ** 4)
    assert tc._a_tview(labels, dims, ["a0", "a1", "a2", "a4", "a5"], ["a3", "a6"]) is None
    # config 5: K = (a0, a3) with the innermost labels free: transposed view
    free = ["a1", "a2", "a4", "a5", "a6"]
    assert tc._a_view(labels, dims, free, ["a0", "a3"]) is None
    ra, rb, srb, kin, ski, ko, sko = tc._a_tview(labels, dims, free, ["a0", "a3"])
    assert (ra, rb, kin, ko) == (4096, 256, 16, 16)
    assert (srb, ski, sko) == (16 ** 4, 16 ** 3, 16 ** 6)
    # config 4: [a0 .. a5] of 32, K = (a1, a5): rows (a0) x (a2 a3 a4)
    labels, dims = [f"a{i}" for i in range(6)], [32] * 6
    v = tc._a_view(labels, dims, ["a0", "a2", "a3", "a4"], ["a1", "a5"])
    assert v == (32, 32768, 32, 32, 32 ** 4, 32, 32 ** 5)
    # K = (a1, a3) with rows (a0) (a2) (a4 a5): three free runs, no view of either kind
    assert tc._a_view(labels, dims, ["a0", "a2", "a4", "a5"], ["a1", "a3"]) is None
    assert tc._a_tview(labels, dims, ["a0", "a2", "a4", "a5"], ["a1", "a3"]) is None
