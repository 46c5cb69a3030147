"""Host-side logic (no GPU): circuits, plans, paths, cost model, records.

Parity is against golden files the reference wrote (tests/golden)."""

from __future__ import annotations

import io
import math

import numpy as np
import pytest

import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import amplitude_engine as ae
from paper_1811_09599_b200 import contraction_plan as cp

CIRCUIT_SPECS = {
    "g4x4_t16_s0": ("grid:4x4", "1+16+1", 0, "cz"),
    "g4x4_t16_s3": ("grid:4x4", "1+16+1", 3, "cz"),
    "g3x4_t16_s11": ("grid:3x4", "1+16+1", 11, "cz"),
    "g3x4_t12_s8": ("grid:3x4", "1+12+1", 8, "cz"),
    "g5x5_t24_s0": ("grid:5x5", "1+24+1", 0, "cz"),
    "g7x7_t40_s0": ("grid:7x7", "1+40+1", 0, "cz"),
    "g7x7_t16_s0": ("grid:7x7", "1+16+1", 0, "cz"),
    "g7x7_t24_s0": ("grid:7x7", "1+24+1", 0, "cz"),
    "b70_t32_s0": ("bristlecone-70", "1+32+1", 0, "cz"),
    "b70_t16_s0": ("bristlecone-70", "1+16+1", 0, "cz"),
    "b70_t24_s0": ("bristlecone-70", "1+24+1", 0, "cz"),
    "b70_t8_s0": ("bristlecone-70", "1+8+1", 0, "cz"),
    "b72_t8_s0": ("bristlecone-72", "1+8+1", 0, "cz"),
    "g2x3_t10_s5_iswap": ("grid:2x3", "1+10+1", 5, "iswap"),
    "g1x2_t8_s1": ("grid:1x2", "1+8+1", 1, "cz"),
    "g2x2_t9_s2": ("grid:2x2", "1+9+1", 2, "cz"),
    "g4x5_t24_s7": ("grid:4x5", "1+24+1", 7, "cz"),
    "g3x3_t0_s4": ("grid:3x3", "1+0+1", 4, "cz"),
}

PLAN_SPECS = {
    "grid4x4_c0": ("grid:4x4", 0), "grid4x4_c1": ("grid:4x4", 1), "grid4x4_c2": ("grid:4x4", 2),
    "grid4x4_def": ("grid:4x4", None), "grid5x5_c1": ("grid:5x5", 1),
    "grid3x4_c1": ("grid:3x4", 1), "grid3x4_c2": ("grid:3x4", 2), "grid3x4_c3": ("grid:3x4", 3),
    "grid2x3_def": ("grid:2x3", None), "grid1x2_def": ("grid:1x2", None),
    "grid2x2_def": ("grid:2x2", None), "grid4x5_def": ("grid:4x5", None),
    "grid3x3_c1": ("grid:3x3", 1),
}


@pytest.mark.parametrize("key", sorted(CIRCUIT_SPECS))
def test_generated_circuits_are_byte_identical(golden, key):
    lat, depth, seed, gate = CIRCUIT_SPECS[key]
    circ = qf.generate_rqc(qf.Lattice.named(lat), depth, seed, two_qubit_gate=gate)
    assert qf.write_circuit(circ) == golden["circuits"][key]


def test_circuit_text_round_trip(golden):
    for text in golden["circuits"].values():
        c = qf.parse_circuit(text)
        assert qf.write_circuit(c) == text


@pytest.mark.parametrize("key", sorted(PLAN_SPECS))
def test_grid_plans_match_reference_text(golden, key):
    lat, n_cuts = PLAN_SPECS[key]
    L = qf.Lattice.named(lat)
    plan = qf.grid_plan(L, n_cuts=n_cuts) if n_cuts is not None else qf.builtin_plan(L)
    assert qf.format_plan(plan) == golden["plans"][key]
    assert qf.format_plan(qf.parse_plan(golden["plans"][key])) == golden["plans"][key]


def test_shipped_slice_plans_match_golden(golden):
    assert qf.format_plan(qf.load_plan("grid:7x7:slice-first")) == golden["plans"]["grid7x7_slice"]
    assert qf.format_plan(qf.load_plan("bristlecone-70:slice-first")) == golden["plans"]["b70_slice"]
    for kind in ("grid:7x7", "bristlecone-70"):
        lat = qf.Lattice.named(kind)
        qf.slice_first_plan(lat).analyze(lat)
        assert qf.format_plan(qf.slice_first_plan(lat)) == \
            qf.format_plan(qf.load_plan(kind + ":slice-first"))


def test_estimate_cost_matches_reference(golden):
    for key, want in golden["costs"].items():
        pkey, ckey = key.split("@")
        circ = qf.parse_circuit(golden["circuits"][ckey])
        plan = qf.parse_plan(golden["plans"][pkey])
        est = qf.estimate_cost(plan, circ.lattice, circ.depth, open_sites=want["open_sites"])
        assert est.paths == want["paths"]
        assert est.total_flops == want["total_flops"]
        assert est.peak_bytes == want["peak_bytes"]
        assert [[s.name, s.flops, s.out_entries, s.evaluations] for s in est.steps] == want["steps"]


def test_reference_path_counts_and_flops_are_consistent(golden):
    """PathStats of the reference equal our symbolic per-amplitude count."""
    case = next(c for c in golden["amplitudes"] if c["name"] == "config2_c64")
    circ = qf.parse_circuit(golden["circuits"][case["circuit"]])
    plan = qf.parse_plan(golden["plans"][case["plan"]])
    est = qf.estimate_cost(plan, circ.lattice, circ.depth)
    assert est.paths == case["paths_total"]
    assert est.total_flops == case["flops"]


class TestEnumeratePaths:
    def test_cartesian(self):
        assert qf.enumerate_paths((2, 3)) == [(i, j) for i in range(2) for j in range(3)]

    def test_fraction_counts(self):
        for f, dims, want in [(0.5, (4, 4), 8), (0.3, (10,), 3), (0.05, (4, 4), 1)]:
            assert len(qf.enumerate_paths(dims, f=f)) == want == math.ceil(f * math.prod(dims))

    def test_seeded_subset(self):
        a = qf.enumerate_paths((4, 4), f=0.5, seed=1)
        assert a == qf.enumerate_paths((4, 4), f=0.5, seed=1)
        assert a != qf.enumerate_paths((4, 4), f=0.5, seed=2)
        assert set(a) <= set(qf.enumerate_paths((4, 4)))
        assert a == sorted(a)

    def test_count_and_errors(self):
        assert len(qf.enumerate_paths((4, 4), count=5)) == 5
        for bad in (0.0, 1.5):
            with pytest.raises(ValueError):
                qf.enumerate_paths((4,), f=bad)
        with pytest.raises(ValueError):
            qf.enumerate_paths((0, 2))

    def test_config5_fraction(self):
        # 16^4 slices at f = 0.005 -> 328 paths
        assert len(qf.enumerate_paths((16, 16, 16, 16), f=0.005, seed=0)) == 328


class TestPlanValidation:
    def lat(self):
        return qf.Lattice.rectangle(2, 2)

    def test_rejects_non_bond_cut(self):
        plan = qf.parse_plan("plan grid:2x2\ncut w 0:3\nloop w\ncontract t0 t1 t2 t3 -> r\noutput r\n")
        with pytest.raises(qf.PlanError):
            plan.analyze(self.lat())

    def test_rejects_cut_use_before_loop(self):
        plan = qf.parse_plan("plan grid:2x2\ncut w 0:1\ncontract t0 t1 -> a\nloop w\n"
                             "contract a t2 t3 -> r\noutput r\n")
        with pytest.raises(qf.PlanError, match="before loop"):
            plan.analyze(self.lat())

    def test_rejects_dangling_and_double_use(self):
        with pytest.raises(qf.PlanError, match="never used"):
            qf.parse_plan("plan grid:2x2\ncontract t0 t1 -> a\ncontract t2 t3 -> r\noutput r\n"
                          ).analyze(self.lat())
        with pytest.raises(qf.PlanError, match="twice"):
            qf.parse_plan("plan grid:2x2\ncontract t0 t1 t1 t2 t3 -> r\noutput r\n"
                          ).analyze(self.lat())

    def test_rejects_bad_reuse_claims(self):
        with pytest.raises(qf.PlanError, match="global"):
            qf.parse_plan("plan grid:2x2\ncut w 0:1\nloop w\ncontract t0 t1 t2 t3 -> r "
                          "reuse=global\noutput r\n").analyze(self.lat())

    def test_parse_errors_carry_line_numbers(self):
        with pytest.raises(qf.PlanError, match="line 2"):
            qf.parse_plan("plan grid:2x2\nbogus x\n")
        with pytest.raises(qf.PlanError, match="header"):
            qf.parse_plan("contract t0 -> r\n")

    def test_cut_values_restrict_dims(self):
        plan = qf.parse_plan("plan grid:2x2\ncut w 0:1 values=0,2\nloop w\n"
                             "contract t0 t1 t2 t3 -> r\noutput r\n")
        assert plan.cut_dims({(0, 1): 4}) == (2,)
        assert cp._decode_bond_values(plan.cuts[0], 1, {(0, 1): 4}) == {(0, 1): 2}

    def test_multi_bond_cut_decoding_msb_first(self):
        cut = qf.CutSpec("w", ((0, 1), (2, 3)))
        assert cp._decode_bond_values(cut, 7, {(0, 1): 4, (2, 3): 4}) == {(0, 1): 1, (2, 3): 3}


def test_memory_budget_escalates_grid_cuts():
    lat = qf.Lattice.rectangle(4, 4)
    base = qf.builtin_plan(lat)
    est = qf.estimate_cost(base, lat, "1+16+1")
    tighter = qf.builtin_plan(lat, "1+16+1", memory_budget=est.peak_bytes - 1)
    assert tighter.num_cuts > base.num_cuts
    with pytest.raises(qf.MemoryBudgetError):
        qf.builtin_plan(lat, "1+16+1", memory_budget=1)


def test_lattice_shapes():
    assert qf.Lattice.named("bristlecone-70").n == 70
    assert qf.Lattice.named("bristlecone-72").n == 72
    lat = qf.Lattice.rectangle(3, 4)
    assert lat.edges()[:3] == ((0, 1), (0, 4), (1, 2))
    assert qf.edge_activations(lat, 8) == {e: 1 for e in lat.edges()}
    assert qf.Lattice.named("bristlecone-24").n == 24
    with pytest.raises(ValueError):
        qf.Lattice.named("bristlecone-23")


def test_circuit_format_errors():
    with pytest.raises(qf.CircuitFormatError):
        qf.parse_circuit("")
    with pytest.raises(qf.CircuitFormatError, match="line 2"):
        qf.parse_circuit("4\n0 foo 1\n")
    with pytest.raises(qf.CircuitFormatError):
        qf.parse_circuit("4\n1 cz 0 3\n")  # not adjacent on 2x2


def test_records_round_trip():
    stats = qf.PathStats(8, 8, 1000, 0)
    batch = qf.AmplitudeBatch("0000", "1010", (2, 3), (0, 3),
                              np.array([1 + 2j, 3 - 1j]), qf.FidelitySpec(), stats)
    assert batch.out_bits(1) == "1011"
    buf = io.StringIO()
    qf.write_amplitudes(buf, qf.batch_records(batch))
    buf.seek(0)
    back = qf.read_amplitudes(buf)
    assert [r["out"] for r in back] == ["1000", "1011"]
    assert back[1]["re"] == 3.0 and back[1]["f_achieved_estimate"] == pytest.approx(160.0)


def test_completions_match_reference_rule():
    assert list(ae._completions(2, 4, 0)) == [0, 1, 2, 3]
    rng = np.random.Generator(np.random.PCG64(5))
    want = np.sort(rng.choice(256, size=32, replace=False))
    assert list(ae._completions(8, 32, 5)) == list(want)


def test_late_bits_validation_and_outs():
    """LateBits host logic (no GPU): the bit matrix contract, the default
    limit (half the batch) and which labels count as open outputs."""
    import torch
    from paper_1811_09599_b200 import tensor_core as tc
    bits = torch.zeros((3, 64), dtype=torch.int32)
    late = tc.LateBits(bits, {"out0": 0, "out2": 2})
    assert (late.nb, late.limit, late.label) == (64, 32, "@b")
    assert tc.LateBits(bits, {}, limit=5).limit == 5
    t = tc.Tensor(("e0_1", "out0", "e0_5", "out2"), torch.zeros(8 * 2 * 8 * 2), (8, 2, 8, 2))
    assert late.outs(t) == ["out0", "out2"]
    assert late._batched_size(t) == 8 * 8 * 64
    with pytest.raises(ValueError):
        tc.LateBits(bits.to(torch.int64), {})
    with pytest.raises(ValueError):
        tc.LateBits(torch.zeros(64, dtype=torch.int32), {})
    with pytest.raises(ValueError):
        tc.LateBits(bits.t(), {})          # not contiguous


def test_contract_shape_counts_open_outputs_like_batch():
    """Per-amplitude flop accounting: batch axes (shared or not) and open
    outputs awaiting a late slice are not part of m or n."""
    import torch
    from paper_1811_09599_b200 import tensor_core as tc
    a = tc.Tensor(("@b", "p", "k"), torch.zeros(4 * 8 * 16), (4, 8, 16))
    b = tc.Tensor(("k", "q", "out3"), torch.zeros(16 * 5 * 2), (16, 5, 2))
    shp = tc.contract_shape(a, b, skip={"out3"})
    assert (shp.batch, shp.m, shp.k, shp.n) == (8, 8, 16, 5)
    assert shp.flops == 8 * 8 * 16 * 5
    assert tc.contract_shape(a, b).n == 10


def test_batch_order_follows_plan_site_order():
    lat = qf.Lattice.rectangle(5, 5)
    circ = qf.generate_rqc(lat, "1+8+1", seed=0)
    eng = qf.AmplitudeEngine(circ, qf.grid_plan(lat, n_cuts=1))
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2, size=(200, 25))
    order = eng.batch_order(bits)
    assert sorted(order.tolist()) == list(range(200))
    seq = []
    for step in eng.plan.steps():
        for x in step.inputs:
            if x.startswith("t") and x[1:].isdigit() and int(x[1:]) not in seq:
                seq.append(int(x[1:]))
    keys = [tuple(row[q] for q in seq) for row in bits[order]]
    assert keys == sorted(keys)


def test_statevector_pass_plan_covers_each_gate_once():
    from paper_1811_09599_b200 import statevector as sv
    lat = qf.Lattice.rectangle(5, 5)
    circ = qf.generate_rqc(lat, "1+8+1", seed=1)
    n = circ.n
    for gates in circ.by_cycle():
        passes = sv.plan_passes(gates, n)
        seen = [g for _, gs in passes for g in gs]
        assert sorted(map(id, seen)) == sorted(map(id, gates))
        for bits, gs in passes:
            assert len(bits) == min(sv.TILE_BITS, n) and bits == sorted(set(bits))
            assert set(range(sv.LOW_BITS)) <= set(bits)
            assert len(gs) <= sv.MAX_OPS
            for g in gs:
                assert {n - 1 - q for q in g.qubits} <= set(bits)


def test_path_groups_split_on_the_other_cuts():
    from paper_1811_09599_b200.amplitude_engine import _path_groups
    paths = [(a, b, c) for a in range(2) for b in range(3) for c in range(2)]
    groups = list(_path_groups(paths, 1))
    # groups vary only cut 1; consecutive paths with other digits equal
    for g in groups:
        assert len({(p[0], p[2]) for p in g}) == 1
    assert sum(len(g) for g in groups) == len(paths)
    assert [len(g) for g in _path_groups([(0, 0), (0, 1), (1, 0), (1, 1)], 1)] == [2, 2]
    assert [len(g) for g in _path_groups([(0,), (1,), (2,)], None)] == [1, 1, 1]


@pytest.mark.parametrize("name,n", [("grid:5x5", 25), ("bristlecone-70", 70)])
def test_batch_order_is_plan_order_lexsort(name, n):
    """The packed-key walk order equals a lexsort over the bits in the order
    the plan first consumes the qubits (ties keep input order)."""
    import numpy as np
    import paper_1811_09599_b200 as qf
    lat = qf.Lattice.named(name)
    circ = qf.generate_rqc(lat, "1+8+1", 0)
    eng = qf.AmplitudeEngine(circ, qf.slice_first_plan(lat) if n == 70 else qf.grid_plan(lat, n_cuts=1))
    bits = np.random.default_rng(1).integers(0, 2, size=(777, n)).astype(np.int32)
    bits[5] = bits[9]                       # a duplicate: stable order
    order = eng.batch_order(bits)
    seq = eng._consume_seq
    assert sorted(seq.tolist()) == list(range(n))
    assert (order == np.lexsort([bits[:, q] for q in reversed(seq)])).all()


def test_permutation_plans_match_reference_moves():
    """plan_permutation keeps the reference's L/R decomposition as plan
    metadata (rq/tensor_core.py:81-206): same moves and fallback on the
    golden cases written by tests/golden/make_golden_moves.py, and the moves
    compose to the permutation."""
    import json
    import os
    from paper_1811_09599_b200 import tensor_core as tcore
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_moves.json")
    with open(path) as fh:
        cases = json.load(fh)
    assert len(cases) >= 400
    for c in cases:
        plan = tcore.plan_permutation(c["dims"], c["perm"], c["mu"], c["nu"])
        assert [[m.kind, list(m.group_perm), m.gamma] for m in plan.moves] == c["moves"], c
        assert plan.fallback == c["fallback"]
        if plan.fallback is None:
            assert tcore.moves_compose(plan) == tuple(c["perm"])
    worked = tcore.plan_permutation([2] * 7, [2, 5, 4, 0, 3, 6, 1], mu=2, nu=4)
    assert worked.move_summary() == [("L", 2), ("R", 4), ("L", 2)]
    with pytest.raises(ValueError):
        tcore.Move("X", (0,), 1)


def test_slice_late_byte_guard():
    """A slice-late step is refused when its open tensor (sliced result x the
    kept cuts' dimensions) would pass the cap or half the memory budget."""
    from types import SimpleNamespace
    lat = qf.Lattice.rectangle(5, 5)
    plan = qf.grid_plan(lat, n_cuts=1)
    from paper_1811_09599_b200.circuits import edge_activations
    from paper_1811_09599_b200.network_builder import edge_label
    bond = {e: 2 ** k for e, k in edge_activations(lat, 24).items() if k > 0}
    tensors = {}
    for s in range(lat.n):
        labels = tuple(sorted(edge_label(*e) for e in bond if s in e))
        dims = tuple(bond[e] for l in labels for e in bond if edge_label(*e) == l)
        tensors[s] = SimpleNamespace(labels=labels, dims=dims, dtype=np.complex64)
    net = SimpleNamespace(tensors=tensors, circuit=SimpleNamespace(lattice=lat), late=None,
                          bond_dim=bond)
    ex = cp.PlanExecutor(net, plan)
    assert ex.late, "config 2 has slice-late steps"
    tight = cp.PlanExecutor(net, plan, memory_budget=1 << 12)
    assert not tight.late
    prev, cp.LATE_OPEN_MAX_BYTES = cp.LATE_OPEN_MAX_BYTES, 16
    try:
        assert not cp.PlanExecutor(net, plan).late
    finally:
        cp.LATE_OPEN_MAX_BYTES = prev
