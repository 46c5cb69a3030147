"""GPU state-vector simulator (complex128) vs the host oracle's state
vector, and the tensor-network engine vs the GPU state vector at config 2's
full size (25 qubits, 1024 bit-strings) -- an independent exact check."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import statevector as sv
from conftest import golden_amps, rel_l2
from oracle import rqc_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("key", ["g3x4_t12_s8", "g4x4_t16_s0"])
@pytest.mark.parametrize("in_bits", [0, 5])
def test_evolve_matches_oracle_state(golden, key, in_bits):
    if key not in golden["circuits"]:
        pytest.skip("no such circuit")
    text = golden["circuits"][key]
    circ = qf.parse_circuit(text)
    got = sv.evolve(circ, in_bits)
    want = O.statevector(text, in_bits)
    assert np.abs(got - want).max() < 1e-12
    assert abs(np.linalg.norm(got) - 1.0) < 1e-12


def test_iswap_circuit_and_tile_sizes():
    lat = qf.Lattice.rectangle(3, 4)
    circ = qf.generate_rqc(lat, "1+8+1", seed=3, two_qubit_gate="iswap")
    want = O.statevector(qf.write_circuit(circ), 0)
    for tb in (5, 7, 10):
        prev, sv.TILE_BITS = sv.TILE_BITS, tb
        try:
            got = sv.evolve(circ, 0)
        finally:
            sv.TILE_BITS = prev
        assert np.abs(got - want).max() < 1e-12


def test_config2_engine_vs_gpu_statevector(golden):
    """All 1024 config-2 amplitudes (5x5, 1+24+1) from the contraction engine
    (late output slicing, CUDA graph) against the exact GPU state vector."""
    case = next(c for c in golden["amplitudes"] if c["name"] == "config2_c64")
    circ = qf.parse_circuit(golden["circuits"][case["circuit"]])
    rng = np.random.Generator(np.random.PCG64(0))
    outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=1024)]
    exact = sv.exact_amplitudes(circ, 0, outs)
    assert rel_l2(exact[:48], golden_amps(case)) < 1e-5
    eng = qf.AmplitudeEngine(circ, qf.parse_plan(golden["plans"][case["plan"]]))
    got, _ = eng.amplitudes(0, outs, graph=True)
    assert rel_l2(got, exact) < 1e-4
    c128 = qf.AmplitudeEngine(circ, qf.parse_plan(golden["plans"][case["plan"]]),
                              dtype=np.complex128)
    got128, _ = c128.amplitudes(0, outs[:64])
    assert rel_l2(got128, exact[:64]) < 1e-10
