"""Frugal rejection sampler (paper_1811_09599_b200.sampler) against the
reference's own outputs (tests/golden/golden_sampler.json, made by
tests/golden/make_golden_sampler.py from rq/sampler.py).  Host logic runs on
CPU; the end-to-end runs (device amplitude batches) are `gpu`."""

from __future__ import annotations

import io
import json

import numpy as np
import pytest

import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import sampler as S


def test_accept_probability_and_required_batches(golden_sampler):
    for m, n_c, p, req in golden_sampler["accept"]:
        assert S.accept_probability(m, n_c) == pytest.approx(p, rel=1e-15)
        assert S.required_batches(m, n_c, 1000) == req
    with pytest.raises(ValueError):
        S.accept_probability(0, 3)
    with pytest.raises(ValueError):
        S.required_batches(10, 3, 0)


def test_frugal_sample_on_probability_arrays_matches_reference(golden_sampler):
    for case in golden_sampler["arrays"]:
        batches = [np.array(b) for b in case["batches"]]
        run = S.frugal_sample(batches, case["m"], case["n"], seed=case["seed"])
        assert list(run.samples) == case["samples"]
        assert run.batches_used == case["batches_used"]
        assert run.tail_mass == pytest.approx(case["tail_mass"], rel=1e-12)
        err = S.estimate_sampling_error(np.concatenate(batches), case["m"], case["n"])
        assert err.epsilon == pytest.approx(case["epsilon"], rel=1e-12)


def test_frugal_sample_stops_and_identities():
    probs = [np.full(4, 0.5), np.full(4, 0.5), np.full(4, 0.5)]
    run = S.frugal_sample(probs, 1, 4, target_samples=2)
    assert run.batches_used == 2 and len(run.samples) == 2
    run = S.frugal_sample([(["a", "b"], [1.0, 0.0])], 1, 2)
    assert run.samples == ("a",)
    assert S.frugal_sample(probs, 1, 4, max_batches=1).batches_used == 1
    with pytest.raises(ValueError):
        S.frugal_sample([np.array([np.nan])], 1, 2)
    with pytest.raises(ValueError):
        S.frugal_sample(probs, 0, 4)
    with pytest.raises(ValueError):
        S.SamplerConfig(n_c=0, target_samples=1)
    with pytest.raises(ValueError):
        S.estimate_sampling_error([], 1, 2)


def test_write_samples_footer():
    run = S.SampleRun(("01", "10"), 3, 2, 10, 4, 6, 0.25)
    fh = io.StringIO()
    S.write_samples(fh, run)
    lines = fh.getvalue().splitlines()
    assert lines[:2] == ["01", "10"]
    foot = json.loads(lines[2])
    assert foot == {"M": 10, "N_C": 2, "batches_used": 3, "acceptance_rate": 2 / 3,
                    "epsilon_estimate": 0.25 * 4 / 6}


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(3))
@pytest.mark.parametrize("group", [1, 5, None])
def test_sample_circuit_matches_reference(golden_sampler, idx, group):
    case = golden_sampler["cases"][idx]
    circ = qf.parse_circuit(case["circuit"])
    eng = qf.AmplitudeEngine(circ, qf.parse_plan(case["plan"]), dtype=np.complex128)
    fid = qf.FidelitySpec(*case["fidelity"])
    cfg = S.SamplerConfig(n_c=case["n_c"], target_samples=case["target"], m=case["m"],
                          seed=case["seed"], fidelity=fid)
    run = S.sample_circuit(eng, case["c_sites"], cfg, group=group)
    assert list(run.samples) == case["samples"]
    assert run.batches_used == case["batches_used"]
    assert run.amplitude_count == case["amplitude_count"]
    assert run.footer()["epsilon_estimate"] == pytest.approx(case["footer"]["epsilon_estimate"],
                                                            rel=1e-8, abs=1e-12)
    stream = S.circuit_batches(eng, case["c_sites"], case["n_c"], seed=case["seed"],
                               fidelity=fid, group=2)
    for want in case["first_batches"]:
        b = next(stream)
        assert b.s_ab == want["s_ab"] and list(b.c_values) == want["c_values"]
        p = np.abs(b.amplitudes) ** 2
        assert np.linalg.norm(p - want["probs"]) <= 1e-10 * np.linalg.norm(want["probs"])
