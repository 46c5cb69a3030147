"""End-to-end parity on the B200: every golden amplitude / batch case the
reference produced, through the product's public API (single, batched,
open-qubit batch), plus the oracle on cases without golden values.

Tolerance: relative L2 <= 1e-4 over each case's amplitude vector for
complex64 (BASELINE.json north_star), 1e-10 for complex128."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1811_09599_b200 as qf
from conftest import golden_amps, rel_l2
from oracle import rqc_oracle as O

pytestmark = pytest.mark.gpu


def _tol(dtype):
    return 1e-10 if dtype == "complex128" else 1e-4


def _engine(golden, case):
    circ = qf.parse_circuit(golden["circuits"][case["circuit"]])
    plan = qf.parse_plan(golden["plans"][case["plan"]])
    return qf.AmplitudeEngine(circ, plan, dtype=np.dtype(case["dtype"]))


def _cases(golden, kind):
    return [c["name"] for c in golden[kind]]


@pytest.fixture(scope="module", params=["auto", "ffma"])
def gemm_mode(request):
    prev = qf.set_gemm_mode(request.param)
    yield request.param
    qf.set_gemm_mode(prev)


@pytest.mark.parametrize("late", [False, True])
@pytest.mark.parametrize("idx", range(19))
def test_amplitude_cases_batched(golden, idx, gemm_mode, late):
    if idx >= len(golden["amplitudes"]):
        pytest.skip("no such case")
    case = golden["amplitudes"][idx]
    eng = _engine(golden, case)
    fid = qf.FidelitySpec(case["f"], case["fseed"])
    got, stats = eng.amplitudes(case["in_bits"], case["out_bits"], fid, late=late)
    assert rel_l2(got, golden_amps(case)) < _tol(case["dtype"]), case["name"]
    assert (stats.paths_total, stats.paths_used, stats.flops) == \
        (case["paths_total"], case["paths_used"], case["flops"])


@pytest.mark.parametrize("idx", range(19))
def test_amplitude_cases_single_call(golden, idx):
    if idx >= len(golden["amplitudes"]):
        pytest.skip("no such case")
    case = golden["amplitudes"][idx]
    eng = _engine(golden, case)
    fid = qf.FidelitySpec(case["f"], case["fseed"])
    outs = case["out_bits"][:3]
    got = []
    for o in outs:
        a, stats = eng.amplitude(case["in_bits"], o, fid)
        got.append(a)
        assert stats.flops == case["flops"]
    want = golden_amps(case)[: len(outs)]
    assert rel_l2(got, want) < _tol(case["dtype"]), case["name"]


@pytest.mark.parametrize("idx", range(8))
def test_batch_cases(golden, idx, gemm_mode):
    if idx >= len(golden["batches"]):
        pytest.skip("no such case")
    case = golden["batches"][idx]
    eng = _engine(golden, case)
    b = eng.amplitude_batch(case["in_bits"], case["s_ab"], case["c_sites"], case["n_c"],
                            seed=case["seed"], fidelity=qf.FidelitySpec(case["f"], case["fseed"]))
    assert list(b.c_values) == case["c_values"]
    assert [b.out_bits(i) for i in range(len(b))] == case["out_bits"]
    assert (b.stats.paths_used, b.stats.flops) == (case["paths_used"], case["flops"])
    assert rel_l2(b.amplitudes, golden_amps(case)) < _tol(case["dtype"]), case["name"]


def test_many_batches_in_one_walk_equal_single_batches(golden):
    case = next(c for c in golden["batches"] if c["name"] == "b70_t16_b64_f64")
    eng = _engine(golden, case)
    rng = np.random.Generator(np.random.PCG64(99))
    sabs = ["".join(str(int(b)) for b in rng.integers(0, 2, size=70)) for _ in range(3)]
    sabs.append(case["s_ab"])
    fid = qf.FidelitySpec(case["f"], case["fseed"])
    many = eng.amplitude_batches(case["in_bits"], sabs, case["c_sites"], 64, seeds=[0] * 4,
                                 fidelity=fid)
    assert rel_l2(many[-1].amplitudes, golden_amps(case)) < 1e-4
    for s, b in zip(sabs, many):
        one = eng.amplitude_batch(case["in_bits"], s, case["c_sites"], 64, seed=0, fidelity=fid)
        assert rel_l2(b.amplitudes, one.amplitudes) < 1e-5


def test_config2_full_1024_bitstrings_vs_oracle(golden):
    """Config 2 as benchmarked: 1024 seeded bit-strings; the first 48 are
    golden (reference), a seeded sample of the rest is checked against the
    oracle."""
    case = next(c for c in golden["amplitudes"] if c["name"] == "config2_c64")
    eng = _engine(golden, case)
    rng = np.random.Generator(np.random.PCG64(0))
    outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=1024)]
    assert outs[:48] == case["out_bits"]
    got, stats = eng.amplitudes(0, outs)
    assert rel_l2(got[:48], golden_amps(case)) < 1e-4
    ora = O.OracleEngine(golden["circuits"][case["circuit"]], golden["plans"][case["plan"]],
                         np.complex128)
    pick = np.random.default_rng(1).choice(1024, size=24, replace=False)
    want = [ora.amplitude(0, outs[i])[0] for i in pick]
    assert rel_l2(got[pick], want) < 1e-4
    # fidelity-estimator sanity: N * mean |a|^2 ~ 1 for a chaotic circuit (f=1)
    est = (2 ** 25) * float(np.mean(np.abs(got) ** 2))
    assert 0.7 < est < 1.3


def test_state_and_cut_identity(golden):
    """Full state vs the double-precision state-vector oracle; the cut sum
    equals the uncut contraction (acceptance C2 analogue)."""
    text = golden["circuits"]["g3x4_t12_s8"]
    circ = qf.parse_circuit(text)
    psi = O.statevector(text, 0)
    for n_cuts in (0, 1, 2, 3):
        eng = qf.AmplitudeEngine(circ, qf.grid_plan(circ.lattice, n_cuts=n_cuts),
                                 dtype=np.complex128)
        assert rel_l2(eng.state(0), psi) < 1e-10
    eng = qf.AmplitudeEngine(circ, qf.grid_plan(circ.lattice, n_cuts=2))
    assert rel_l2(eng.state(0), psi) < 1e-4


def test_reuse_cache_is_transparent(golden):
    circ = qf.parse_circuit(golden["circuits"]["g4x4_t16_s3"])
    plan = qf.grid_plan(circ.lattice, n_cuts=2)
    eng = qf.AmplitudeEngine(circ, plan, dtype=np.complex128)
    net = eng.base_net(0).fix_outputs({q: 0 for q in range(16)})
    dims = plan.cut_dims(net.bond_dim)
    paths = qf.enumerate_paths(dims)
    with_cache = sum(qf.execute_plan(net, plan, p).scalar() for p in paths)
    ex = qf.PlanExecutor(net, plan, enable_reuse=False)
    without = sum(ex.run(p).scalar() for p in paths)
    assert abs(with_cache - without) < 1e-12


def test_memory_budget_and_errors(golden):
    circ = qf.parse_circuit(golden["circuits"]["g4x4_t16_s0"])
    eng = qf.AmplitudeEngine(circ, qf.grid_plan(circ.lattice, 1), memory_budget=1024)
    with pytest.raises(qf.MemoryBudgetError):
        eng.amplitude(0, 5)
    eng = qf.AmplitudeEngine(circ)
    with pytest.raises(ValueError):
        eng.amplitude(0, 2 ** 16)
    with pytest.raises(ValueError):
        eng.amplitude_batch(0, 0, (14, 15), 5)
    with pytest.raises(ValueError):
        eng.amplitude_batch(0, 0, (), 1)


def test_nonzero_input_and_bristlecone72_fold(golden):
    text = golden["circuits"]["b72_t8_s0"]
    circ = qf.parse_circuit(text)
    # the 72-site frame folds its two corners into their neighbours
    eng = qf.AmplitudeEngine(circ, qf.load_plan("bristlecone-70").__class__(
        "bristlecone-72", (), (("contract", qf.ContractStep(
            tuple(f"t{s}" for s in range(72) if s not in (0, 71)), "r", None)), ("output", "r")),
        ()))
    net = eng.base_net(0)
    assert sorted(net.tensors) == [s for s in range(72) if s not in (0, 71)]


def test_slice_late_is_transparent(golden):
    """Slice-late execution (cut bonds left open in steps whose cut
    dependence enters only through their own site tensors) gives the same
    amplitudes and the same reference flop count as slicing early."""
    case = next(c for c in golden["amplitudes"] if c["name"] == "config2_c64")
    circ = qf.parse_circuit(golden["circuits"][case["circuit"]])
    plan = qf.parse_plan(golden["plans"][case["plan"]])
    eng = qf.AmplitudeEngine(circ, plan)
    outs = case["out_bits"][:16]
    bits = np.array([[int(c) for c in o] for o in outs], dtype=np.int32)
    net = eng.base_net(0).fix_outputs_batch(bits, tuple(range(circ.n)))
    res = {}
    for late in (True, False):
        ex = qf.PlanExecutor(net, plan, slice_late=late)
        if late:
            assert set(ex.late) == {"A", "B"}
        tot = None
        for p in qf.enumerate_paths(ex.cut_dims):
            r = ex.run(p).data.clone()
            tot = r if tot is None else tot + r
        res[late] = (tot.cpu().numpy(), ex.flops)
    assert rel_l2(res[True][0], res[False][0]) < 1e-6
    assert res[True][1] == res[False][1] == case["flops"]
    assert rel_l2(res[True][0], golden_amps(case)[:16]) < 1e-4


@pytest.mark.parametrize("late", [False, True])
@pytest.mark.parametrize("name", ["config1_c64", "config2_c64", "g4x4s3_cuts2_f025_c64"])
def test_cuda_graph_replay_matches_eager(golden, name, late):
    case = next(c for c in golden["amplitudes"] if c["name"] == name)
    eng = _engine(golden, case)
    fid = qf.FidelitySpec(case["f"], case["fseed"])
    outs = case["out_bits"]
    eager, st_e = eng.amplitudes(case["in_bits"], outs, fid, late=not late)
    for _ in range(2):  # capture once, then replay with new bits each call
        g1, st_g = eng.amplitudes(case["in_bits"], outs, fid, graph=True, late=late)
        assert rel_l2(g1, eager) < 1e-6
        assert (st_g.flops, st_g.paths_used) == (st_e.flops, st_e.paths_used)
    rev = list(reversed(outs))
    g2, _ = eng.amplitudes(case["in_bits"], rev, fid, graph=True, late=late)
    assert rel_l2(g2, eager[::-1]) < 1e-6
    assert rel_l2(g1, golden_amps(case)) < 1e-4


@pytest.mark.parametrize("limit", [1, 2, 16, 2 ** 16])
@pytest.mark.parametrize("name", ["config1_c64", "g4x4s3_cuts2_f025_c64", "config1_c128"])
def test_late_output_slicing_limits(golden, name, limit):
    """Late output slicing at every threshold: limit 1 slices at the first
    contraction, 2^16 keeps a 4x4 network fully open (the whole output state
    is contracted, then the bit-strings are sliced from it)."""
    case = next((c for c in golden["amplitudes"] if c["name"] == name), None)
    if case is None:
        pytest.skip("no such case")
    eng = _engine(golden, case)
    fid = qf.FidelitySpec(case["f"], case["fseed"])
    n = eng.circuit.n
    bits = np.array([[int(ch) for ch in o] for o in case["out_bits"]], dtype=np.int32)
    base = eng.base_net(case["in_bits"])
    bits_t = torch.from_numpy(np.ascontiguousarray(bits.T)).cuda()
    net = base.late_outputs(bits_t, tuple(range(n)), limit=limit)
    ex = eng._executor(net)
    from paper_1811_09599_b200.amplitude_engine import _finisher
    fin = _finisher(net)
    tot = None
    for p in fid.paths_for(ex.cut_dims):
        r = fin(ex.run(p))
        tot = r.clone() if tot is None else tot + r
    assert rel_l2(tot.cpu().numpy()[: len(bits)], golden_amps(case)) < _tol(case["dtype"])
    assert ex.flops == case["flops"]


def test_late_config2_1024_matches_early(golden):
    case = next(c for c in golden["amplitudes"] if c["name"] == "config2_c64")
    eng = _engine(golden, case)
    rng = np.random.Generator(np.random.PCG64(0))
    outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=1024)]
    early, st0 = eng.amplitudes(0, outs, late=False)
    late, st1 = eng.amplitudes(0, outs, late=True)
    assert rel_l2(late, early) < 1e-5
    assert (st0.flops, st0.paths_used) == (st1.flops, st1.paths_used)
    assert rel_l2(late[:48], golden_amps(case)) < 1e-4


@pytest.mark.parametrize("late", [False, True])
@pytest.mark.parametrize("idx", range(19))
def test_path_batching_is_transparent(golden, idx, late):
    """Walking all values of the last cut as one batched pass (the value an
    extra batch index, operands without it broadcast) gives the per-path
    walk's amplitudes and exactly the reference's PathStats."""
    if idx >= len(golden["amplitudes"]):
        pytest.skip("no such case")
    case = golden["amplitudes"][idx]
    eng = _engine(golden, case)
    fid = qf.FidelitySpec(case["f"], case["fseed"])
    from paper_1811_09599_b200 import amplitude_engine as ae
    prev = qf.set_path_batching(False)
    try:
        ref, st0 = eng.amplitudes(case["in_bits"], case["out_bits"], fid, late=late)
    finally:
        qf.set_path_batching(prev)
    qf.set_path_batching(True)
    n0 = ae.PATH_GROUPS_RUN[0]
    got, st1 = eng.amplitudes(case["in_bits"], case["out_bits"], fid, late=late)
    single, _ = eng.amplitude(case["in_bits"], case["out_bits"][0], fid)
    qf.set_path_batching(prev)
    assert rel_l2(got, ref) < 1e-5, case["name"]
    assert rel_l2(got, golden_amps(case)) < _tol(case["dtype"]), case["name"]
    assert abs(single - golden_amps(case)[0]) <= _tol(case["dtype"]) * 10 * \
        max(abs(golden_amps(case)[0]), np.linalg.norm(golden_amps(case)) / len(got))
    assert (st1.paths_total, st1.paths_used, st1.flops) == \
        (case["paths_total"], case["paths_used"], case["flops"])
    if case["name"].startswith("config2") and late and case["dtype"] == "complex64":
        assert ae.PATH_GROUPS_RUN[0] > n0, "config 2 should walk its cut values as one group"
