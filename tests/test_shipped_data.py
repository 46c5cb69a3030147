"""Drop-in data parity: every Bristlecone lattice and every shipped plan of
the reference (rq/circuits.py:130-170, rq/contraction_plan.py:778-821)
through the product's public API, against tests/golden/golden_shipped.json
(written by tests/golden/make_golden_shipped.py from rqcsim itself)."""

from __future__ import annotations

import json
import os

import pytest

import paper_1811_09599_b200 as qf
from conftest import GOLDEN


@pytest.fixture(scope="module")
def shipped():
    with open(os.path.join(GOLDEN, "golden_shipped.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("size", qf.circuits.BRISTLECONE_SIZES)
def test_bristlecone_lattices_equal_reference(shipped, size):
    want = shipped["lattices"][str(size)]
    lat = qf.Lattice.named(f"bristlecone-{size}")
    assert lat.n == size
    assert [list(x) for x in lat.sites] == want["sites"]
    assert [list(e) for e in lat.edges()] == want["edges"]


def test_unknown_bristlecone_size_raises():
    with pytest.raises(ValueError):
        qf.Lattice.named("bristlecone-25")


@pytest.mark.parametrize("name", sorted(qf.shipped_plans()))
def test_builtin_plans_are_the_reference_plans(shipped, name):
    assert name in shipped["plans"]
    lat = qf.Lattice.named(name)
    plan = qf.builtin_plan(lat)
    assert qf.format_plan(plan) == qf.format_plan(qf.parse_plan(shipped["plans"][name]))
    assert qf.format_plan(qf.load_plan(name)) == qf.format_plan(plan)
    plan.analyze(lat)
    for depth in ("1+8+1", "1+16+1"):
        want = shipped["costs"][f"{name} {depth}"]
        est = qf.estimate_cost(plan, lat, depth)
        assert (est.total_flops, est.peak_bytes, est.paths) == \
            (want["flops"], want["peak_bytes"], want["paths"])


def test_shipped_plans_fail_a_memory_budget_at_full_depth():
    lat = qf.Lattice.named("grid:7x7")
    with pytest.raises(qf.MemoryBudgetError):
        qf.builtin_plan(lat, "1+40+1", memory_budget=180 * 2 ** 30)
    est = qf.estimate_cost(qf.slice_first_plan(lat), lat, "1+40+1")
    assert est.peak_bytes < 80 * 2 ** 30


@pytest.mark.parametrize("size", [24, 48, 60])
def test_bristlecone_circuits_generate_and_plan(size):
    lat = qf.Lattice.named(f"bristlecone-{size}")
    circ = qf.generate_rqc(lat, "1+8+1", 0)
    assert qf.parse_circuit(qf.write_circuit(circ)).n == size
    qf.builtin_plan(lat).analyze(lat)
