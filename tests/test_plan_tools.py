"""Plan tooling on the CPU: path-subset flop counts
against the reference's PathStats in the golden fixtures, and greedy
reordering / budgeted slicing checked for cost and (through the numpy
oracle, test infrastructure) for unchanged amplitudes."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import plan_tools as pt
from conftest import rel_l2
from oracle import rqc_oracle as O


def _golden_case(golden, name):
    return next(c for c in golden["amplitudes"] if c["name"] == name)


@pytest.mark.parametrize("idx", range(17))
def test_path_subset_flops_match_reference_pathstats(golden, idx):
    case = golden["amplitudes"][idx]
    circ = qf.parse_circuit(golden["circuits"][case["circuit"]])
    plan = qf.parse_plan(golden["plans"][case["plan"]])
    if any(g.name == "iswap" for g in circ.gates):
        pytest.skip("iSWAP bonds: the reference's dimension quirk (DESIGN §5)")
    lat = circ.lattice
    got = pt.fidelity_flops(plan, lat, circ.depth, case["f"], case["fseed"])
    assert got == case["flops"], case["name"]


def test_full_path_list_equals_estimate_cost():
    lat = qf.Lattice.named("grid:5x5")
    plan = qf.grid_plan(lat, n_cuts=2)
    est = qf.estimate_cost(plan, lat, "1+24+1")
    dims = plan.cut_dims(pt.bond_dims(lat, "1+24+1"))
    assert pt.path_subset_flops(plan, lat, "1+24+1", qf.enumerate_paths(dims)) == est.total_flops


def test_shard_flops_add_up():
    """Contiguous shards (slices.shard_range) re-execute only the shared
    prefix steps: the sum over shards >= the single walk."""
    lat = qf.Lattice.named("grid:4x4")
    plan = qf.grid_plan(lat, n_cuts=2)
    dims = plan.cut_dims(pt.bond_dims(lat, "1+16+1"))
    paths = qf.enumerate_paths(dims)
    whole = pt.path_subset_flops(plan, lat, "1+16+1", paths)
    from paper_1811_09599_b200.slices import shard_range
    parts = 0
    for r in range(4):
        lo, hi = shard_range(len(paths), r, 4)
        parts += pt.path_subset_flops(plan, lat, "1+16+1", paths[lo:hi])
    assert parts >= whole


@pytest.mark.parametrize("shape,depth", [("grid:4x4", "1+16+1"), ("grid:5x5", "1+24+1"),
                                         ("grid:4x5", "1+20+1")])
def test_reorder_never_costs_more(shape, depth):
    lat = qf.Lattice.named(shape)
    for n_cuts in (0, 1):
        plan = qf.grid_plan(lat, n_cuts=n_cuts)
        new = pt.reorder_plan(plan, lat, depth)
        a = qf.estimate_cost(plan, lat, depth).total_flops
        b = qf.estimate_cost(new, lat, depth).total_flops
        assert b <= a
        assert [s.name for s in new.steps()] == [s.name for s in plan.steps()]
        assert sorted(new.site_ids()) == sorted(plan.site_ids())


def test_reordered_plan_same_amplitudes_oracle():
    lat = qf.Lattice.named("grid:3x4")
    circ = qf.generate_rqc(lat, "1+8+1", seed=3)
    plan = qf.grid_plan(lat, n_cuts=1)
    new = pt.reorder_plan(plan, lat, "1+8+1")
    text = qf.write_circuit(circ)
    outs = ["010011010110", "111100001010", "000000000001"]
    a = [O.OracleEngine(text, qf.format_plan(plan), np.complex128).amplitude(0, o)[0] for o in outs]
    b = [O.OracleEngine(text, qf.format_plan(new), np.complex128).amplitude(0, o)[0] for o in outs]
    assert rel_l2(b, a) < 1e-10


def test_slice_for_budget_fits_and_keeps_amplitudes():
    lat = qf.Lattice.named("grid:3x4")
    depth = "1+16+1"
    circ = qf.generate_rqc(lat, depth, seed=1)
    base = qf.grid_plan(lat, n_cuts=0)
    region_c = set(base.batch_sites)
    ab = sorted(set(range(lat.n)) - region_c)
    region_a = {s for s in ab if lat.coords(s)[1] < 2}
    region_b = set(ab) - region_a
    full = qf.estimate_cost(qf.two_region_plan(lat, region_a, region_b, region_c, []), lat, depth)
    budget = full.peak_bytes // 2
    plan = pt.slice_for_budget(lat, depth, region_a, region_b, region_c, budget)
    est = qf.estimate_cost(plan, lat, depth)
    assert est.peak_bytes <= budget and plan.num_cuts >= 1
    text = qf.write_circuit(circ)
    outs = ["010011010110", "101100001011"]
    ref = qf.grid_plan(lat, n_cuts=0)
    a = [O.OracleEngine(text, qf.format_plan(ref), np.complex128).amplitude(0, o)[0] for o in outs]
    b = [O.OracleEngine(text, qf.format_plan(plan), np.complex128).amplitude(0, o)[0] for o in outs]
    assert rel_l2(b, a) < 1e-10


def test_slice_for_budget_impossible_raises():
    lat = qf.Lattice.named("grid:3x3")
    with pytest.raises(qf.PlanError):
        pt.slice_for_budget(lat, "1+8+1", {0, 1, 3, 4}, {2, 5}, {6, 7, 8}, 1, max_cuts=1)


# ---------------------------------------------------------------------------
# exact subset-DP trees (plan_tools.tree_order / tree_plan)

_D_REGION = [24, 25, 26, 27, 31, 32, 33, 34, 38, 39, 40, 41, 45, 46, 47, 48]


def _max_lg_of_chain(lat, order, bonds, sliced):
    acc, worst, flops = None, 0, 0
    for s in order:
        op = pt._site_shape(lat, s, bonds, sliced, set())
        if acc is None:
            acc = op
            continue
        f, acc = pt._fold_cost(acc, op)
        flops += f
        worst = max(worst, sum(pt._lg(d) for d in acc.values()))
    return flops, worst


def test_tree_order_rediscovers_7x7_region_d_tree():
    """Region D of the 7x7 (1+40+1) plan: the exact DP finds a tree with every
    intermediate <= 2^30 at 4.48e13 flops, where the
    reference's greedy region order (rq/contraction_plan.py:651-673) peaks
    above 2^30 and costs more."""
    from paper_1811_09599_b200.contraction_plan import _region_order
    from paper_1811_09599_b200.network_builder import edge_label
    lat = qf.Lattice.named("grid:7x7")
    bonds = pt.bond_dims(lat, "1+40+1")
    sliced = {edge_label(19, 26), edge_label(37, 38)}
    flops, tree = pt.tree_order(lat, _D_REGION, bonds, sliced=sliced, cap_log2=30)
    assert sorted(pt._tree_sites(tree)) == _D_REGION
    assert flops <= 4.49e13
    g_flops, g_worst = _max_lg_of_chain(lat, _region_order(lat, _D_REGION), bonds, sliced)
    assert g_worst > 30 and g_flops > flops


def test_tree_plan_7x7_matches_or_beats_the_hand_slice_first_plan():
    lat = qf.Lattice.named("grid:7x7")
    plan = pt.tree_plan(qf.load_plan("grid:7x7"), lat, "1+40+1")
    plan.analyze(lat)
    est = qf.estimate_cost(plan, lat, "1+40+1")
    hand = qf.estimate_cost(qf.slice_first_plan(lat), lat, "1+40+1")
    shipped = qf.estimate_cost(qf.load_plan("grid:7x7"), lat, "1+40+1")
    assert est.total_flops <= hand.total_flops
    assert est.peak_bytes < 80 * 2 ** 30 < shipped.peak_bytes
    assert [c.name for c in plan.cuts] == ["right", "bottom"]
    assert plan.batch_sites == qf.load_plan("grid:7x7").batch_sites


@pytest.mark.parametrize("name,cap,peak_gib", [("bristlecone-48", 30, 32), ("bristlecone-60", 32, 80),
                                               ("bristlecone-64", 32, 64), ("bristlecone-70", 30, 32)])
def test_tree_plans_for_bristlecone_are_feasible_at_full_depth(name, cap, peak_gib):
    """Bris-48/60/64/70 at 1+32+1 with their shipped cuts: the shipped plans
    need 10^4..10^11 GiB; the tree plans fit a B200."""
    lat = qf.Lattice.named(name)
    ship = qf.load_plan(name)
    c_sites = tuple(sorted(ship.batch_sites[:6]))
    plan = pt.tree_plan(ship, lat, "1+32+1", open_sites=c_sites, cap_log2=cap)
    est = qf.estimate_cost(plan, lat, "1+32+1", open_sites=c_sites)
    est0 = qf.estimate_cost(ship, lat, "1+32+1", open_sites=c_sites)
    assert est.peak_bytes < peak_gib * 2 ** 30 < est0.peak_bytes
    assert est.total_flops < est0.total_flops


@pytest.mark.parametrize("name,depth", [("grid:7x7", "1+16+1"), ("bristlecone-48", "1+8+1"),
                                        ("bristlecone-24", "1+8+1")])
def test_tree_plan_amplitudes_equal_shipped_plan(name, depth):
    """Same amplitudes as the shipped plan (numpy oracle, test infrastructure)."""
    lat = qf.Lattice.named(name)
    circ = qf.generate_rqc(lat, depth, 3)
    ship = qf.load_plan(name)
    tree = pt.tree_plan(ship, lat, depth)
    text = qf.write_circuit(circ)
    a = O.OracleEngine(text, qf.format_plan(ship), np.complex128)
    b = O.OracleEngine(text, qf.format_plan(tree), np.complex128)
    rng = np.random.default_rng(4)
    for _ in range(2):
        out = "".join(str(int(x)) for x in rng.integers(0, 2, size=lat.n))
        assert abs(a.amplitude(0, out)[0] - b.amplitude(0, out)[0]) <= 1e-10 * abs(a.amplitude(0, out)[0])
