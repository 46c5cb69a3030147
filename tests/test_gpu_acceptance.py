"""The reference's acceptance criterion 6 (pkg/tests/test_acceptance.py:
271-305) through the product: an open-qubit batch agrees with single
amplitudes, and a 32-entry batch costs at most 1.5x one single amplitude
(fresh engine per timed call, median of 7)."""

from __future__ import annotations

import time

import numpy as np
import pytest
import torch

import paper_1811_09599_b200 as qf

pytestmark = pytest.mark.gpu


def test_criterion_06_batch_consistency_and_cost():
    lat = qf.Lattice.named("bristlecone-24")
    circ = qf.generate_rqc(lat, "1+16+1", seed=1)
    plan = qf.builtin_plan(lat, "1+16+1")
    c_sites = plan.batch_sites
    eng = qf.AmplitudeEngine(circ, dtype=np.complex128)
    batch = eng.amplitude_batch(0, 0, c_sites, 32, seed=4)
    worst = 0.0
    for i in range(32):
        single, _ = eng.amplitude(0, batch.out_bits(i))
        worst = max(worst, abs(batch.amplitudes[i] - single))
    assert worst <= 1e-6

    def timed(fn, repeats=7):
        samples = []
        for _ in range(repeats):
            fresh = qf.AmplitudeEngine(circ, dtype=np.complex128)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(fresh)
            torch.cuda.synchronize()
            samples.append(time.perf_counter() - t0)
        return float(np.median(samples))

    t_one = timed(lambda e: e.amplitude(0, 0))
    t_batch = timed(lambda e: e.amplitude_batch(0, 0, c_sites, 32, seed=4))
    assert t_batch / t_one <= 1.5, (t_batch, t_one)


def test_single_amplitude_calls_match_batched_config2(golden):
    """The drop-in single-call API (rq/amplitude_engine.py:114-126) on the
    config-2 circuit: repeated calls reuse the cached network and executor
    state and agree with the batched walk."""
    case = next(c for c in golden["amplitudes"] if c["name"] == "config2_c64")
    circ = qf.parse_circuit(golden["circuits"][case["circuit"]])
    eng = qf.AmplitudeEngine(circ, qf.parse_plan(golden["plans"][case["plan"]]))
    got = np.array([eng.amplitude(case["in_bits"], o)[0] for o in case["out_bits"][:16]])
    batched, _ = eng.amplitudes(case["in_bits"], case["out_bits"][:16])
    assert np.linalg.norm(got - batched) <= 1e-5 * np.linalg.norm(batched)
