"""Pin the CPU oracle (oracle/rqc_oracle.py) against the reference's own
outputs (tests/golden/*.json, produced by tests/golden/make_golden.py)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_amps, rel_l2
from oracle import rqc_oracle as O


def _tol(dtype):
    return 1e-10 if dtype == "complex128" else 2e-5


def test_lattices_match_circuit_headers(golden):
    for key, text in golden["circuits"].items():
        c = O.parse_circuit(text)
        assert c.n == len(c.sites)
        # every two-qubit gate must sit on a lattice edge
        edges = set(c.edges)
        for _, _, qs in c.gates:
            if len(qs) == 2:
                assert tuple(sorted(qs)) in edges, key


@pytest.mark.parametrize("idx", range(19))
def test_oracle_amplitudes_match_reference(golden, idx):
    cases = golden["amplitudes"]
    if idx >= len(cases):
        pytest.skip("no such case")
    case = cases[idx]
    eng = O.OracleEngine(golden["circuits"][case["circuit"]], golden["plans"][case["plan"]],
                         dtype=np.dtype(case["dtype"]))
    got = []
    for ob in case["out_bits"]:
        a, ptot, pused, flops = eng.amplitude(case["in_bits"], ob, case["f"], case["fseed"])
        got.append(a)
        assert (ptot, pused, flops) == (case["paths_total"], case["paths_used"], case["flops"])
    assert rel_l2(got, golden_amps(case)) < _tol(case["dtype"]), case["name"]


@pytest.mark.parametrize("idx", range(8))
def test_oracle_batches_match_reference(golden, idx):
    cases = golden["batches"]
    if idx >= len(cases):
        pytest.skip("no such case")
    case = cases[idx]
    if case["name"].startswith("b70_t24"):
        pytest.skip("slow on CPU; covered by the GPU parity test")
    eng = O.OracleEngine(golden["circuits"][case["circuit"]], golden["plans"][case["plan"]],
                         dtype=np.dtype(case["dtype"]))
    vals, amps, flops, pused = eng.amplitude_batch(case["in_bits"], case["s_ab"], case["c_sites"],
                                                   case["n_c"], case["seed"], case["f"], case["fseed"])
    assert list(vals) == case["c_values"]
    assert (flops, pused) == (case["flops"], case["paths_used"])
    assert rel_l2(amps, golden_amps(case)) < _tol(case["dtype"]), case["name"]


def test_oracle_permutation_bytes_match_reference(golden_perm):
    for case in golden_perm["cases"]:
        g = np.random.default_rng(case["input_seed"])
        dims = case["dims"]
        x = (g.standard_normal(dims) + 1j * g.standard_normal(dims)).astype(np.complex64)
        y = O.permute_naive(x, case["perm"])
        assert hashlib.sha256(y.tobytes()).hexdigest() == case["sha256"]


def test_statevector_oracle_agrees_with_golden(golden):
    case = next(c for c in golden["amplitudes"] if c["name"] == "config1_c128")
    psi = O.statevector(golden["circuits"][case["circuit"]], 0)
    got = [psi[int(b, 2)] for b in case["out_bits"]]
    assert rel_l2(got, golden_amps(case)) < 1e-10


def test_c_permutation_oracle_matches_reference_bytes(golden_perm):
    """oracle/permute_ref.c reproduces the reference's permute_fast bytes."""
    import hashlib
    from oracle import permute_oracle as P
    for case in golden_perm["cases"]:
        g = np.random.default_rng(case["input_seed"])
        dims = case["dims"]
        x = (g.standard_normal(dims) + 1j * g.standard_normal(dims)).astype(np.complex64)
        out = P.permute(x, dims, case["perm"])
        assert hashlib.sha256(out.tobytes()).hexdigest() == case["sha256"], case
