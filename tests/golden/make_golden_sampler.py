"""Golden fixtures for the frugal rejection sampler, made by importing the
REFERENCE implementation (rq/sampler.py) in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \\
        python tests/golden/make_golden_sampler.py

Writes tests/golden/golden_sampler.json: for seeded small circuits, the
reference's `sample_circuit` output (accepted bit-strings, footer), the
first batches of its `circuit_batches` stream (s_AB, completions,
probabilities), and `frugal_sample`/`estimate_sampling_error` on fixed
probability arrays.  Only the committed JSON is used at test time.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from rqcsim import (AmplitudeEngine, FidelitySpec, Lattice, format_plan,  # noqa: E402
                    generate_rqc, grid_plan, write_circuit)
from rqcsim import sampler as S  # noqa: E402


def run_case(name, rows, cols, depth, seed, n_cuts, c_sites, n_c, m, target, fid, sseed):
    lat = Lattice.rectangle(rows, cols)
    circ = generate_rqc(lat, depth, seed)
    plan = grid_plan(lat, n_cuts=n_cuts)
    eng = AmplitudeEngine(circ, plan, dtype=np.complex128)
    cfg = S.SamplerConfig(n_c=n_c, target_samples=target, m=m, seed=sseed,
                          fidelity=FidelitySpec(*fid))
    run = S.sample_circuit(eng, c_sites, cfg)
    stream = S.circuit_batches(eng, c_sites, n_c, seed=sseed, fidelity=FidelitySpec(*fid))
    first = []
    for _ in range(3):
        b = next(stream)
        first.append({"s_ab": b.s_ab, "c_values": list(b.c_values),
                      "probs": [float(abs(a) ** 2) for a in b.amplitudes]})
    return {"name": name, "circuit": write_circuit(circ), "plan": format_plan(plan),
            "c_sites": list(c_sites), "n_c": n_c, "m": m, "target": target, "seed": sseed,
            "fidelity": list(fid), "samples": list(run.samples), "footer": run.footer(),
            "batches_used": run.batches_used, "amplitude_count": run.amplitude_count,
            "tail_mass": run.tail_mass, "first_batches": first}


def main():
    cases = [
        run_case("g4x4_t8_nc16", 4, 4, "1+8+1", 0, 0, (10, 11, 14, 15), 16, 10, 12, (1.0, 0), 0),
        run_case("g4x4_t12_nc8_cut", 4, 4, "1+12+1", 2, 1, (0, 1, 4), 8, 4, 10, (1.0, 0), 7),
        run_case("g3x4_t8_nc5_f05", 3, 4, "1+8+1", 1, 1, (8, 9, 10, 11), 5, 6, 8, (0.5, 3), 11),
    ]
    rng = np.random.Generator(np.random.PCG64(5))
    arrays = []
    for size, count in ((4, 6), (30, 10)):
        batches = [rng.exponential(1.0, size=size) / 2 ** 10 for _ in range(count)]
        run = S.frugal_sample([b.copy() for b in batches], 10, 2 ** 10, seed=3)
        err = S.estimate_sampling_error(np.concatenate(batches), 10, 2 ** 10)
        arrays.append({"batches": [b.tolist() for b in batches], "m": 10, "n": 2 ** 10, "seed": 3,
                       "samples": list(run.samples), "batches_used": run.batches_used,
                       "tail_mass": run.tail_mass, "epsilon": err.epsilon})
    out = {"cases": cases, "arrays": arrays,
           "accept": [[m, n_c, S.accept_probability(m, n_c), S.required_batches(m, n_c, 1000)]
                      for m, n_c in ((10, 30), (4, 8), (1, 1), (20, 64))]}
    with open(os.path.join(HERE, "golden_sampler.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", len(cases), "circuit cases")


if __name__ == "__main__":
    main()
