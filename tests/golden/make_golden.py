"""Generate the golden fixtures by importing the REFERENCE implementation.

Run once in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It writes tests/golden/golden.json (+ golden_perm.json).  Everything in
there is an output of the reference package `rqcsim`
(/root/reference/pkg/src/rqcsim): circuit files from `generate_rqc` +
`write_circuit`, plan files from `grid_plan`/`format_plan`, amplitudes
and PathStats from `AmplitudeEngine.amplitude`/`.amplitude_batch`,
symbolic costs from `estimate_cost`, and permutation bytes from
`permute_fast`.  The product's slice-first plans
(paper_1811_09599_b200/data/plans/*_slice.txt) are executed by the
reference's own executor at reduced depth.  Nothing here is used at run
time on the GPU box except the committed JSON.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
PLANS = os.path.join(REPO, "paper_1811_09599_b200", "data", "plans")

sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from rqcsim import (AmplitudeEngine, FidelitySpec, Lattice,  # noqa: E402
                    estimate_cost, format_plan, generate_rqc, grid_plan,
                    parse_plan, write_circuit)
from rqcsim.contraction_plan import builtin_plan  # noqa: E402
from rqcsim.tensor_core import permute_fast, permute_naive, plan_permutation  # noqa: E402

CIRCUITS = [
    # key, lattice, depth, seed, two-qubit gate
    ("g4x4_t16_s0", "grid:4x4", "1+16+1", 0, "cz"),      # config 1
    ("g4x4_t16_s3", "grid:4x4", "1+16+1", 3, "cz"),
    ("g3x4_t16_s11", "grid:3x4", "1+16+1", 11, "cz"),
    ("g3x4_t12_s8", "grid:3x4", "1+12+1", 8, "cz"),
    ("g5x5_t24_s0", "grid:5x5", "1+24+1", 0, "cz"),      # config 2
    ("g7x7_t40_s0", "grid:7x7", "1+40+1", 0, "cz"),      # config 4 (text only)
    ("g7x7_t16_s0", "grid:7x7", "1+16+1", 0, "cz"),      # config 4 reduced depth
    ("b70_t32_s0", "bristlecone-70", "1+32+1", 0, "cz"),  # config 5 (text only)
    ("b70_t16_s0", "bristlecone-70", "1+16+1", 0, "cz"),  # config 5 reduced depth
    ("b70_t8_s0", "bristlecone-70", "1+8+1", 0, "cz"),
    ("g7x7_t24_s0", "grid:7x7", "1+24+1", 0, "cz"),      # config 4 at bond 8
    ("b70_t24_s0", "bristlecone-70", "1+24+1", 0, "cz"),  # config 5 at bond 8
    ("b72_t8_s0", "bristlecone-72", "1+8+1", 0, "cz"),
    ("g2x3_t10_s5_iswap", "grid:2x3", "1+10+1", 5, "iswap"),
    ("g1x2_t8_s1", "grid:1x2", "1+8+1", 1, "cz"),
    ("g2x2_t9_s2", "grid:2x2", "1+9+1", 2, "cz"),
    ("g4x5_t24_s7", "grid:4x5", "1+24+1", 7, "cz"),
    ("g3x3_t0_s4", "grid:3x3", "1+0+1", 4, "cz"),
]

GRID_PLANS = [
    # key, lattice, n_cuts (None = builtin default)
    ("grid4x4_c0", "grid:4x4", 0),   # config 1
    ("grid4x4_c1", "grid:4x4", 1),
    ("grid4x4_c2", "grid:4x4", 2),
    ("grid4x4_def", "grid:4x4", None),
    ("grid5x5_c1", "grid:5x5", 1),   # config 2
    ("grid3x4_c1", "grid:3x4", 1),
    ("grid3x4_c2", "grid:3x4", 2),
    ("grid3x4_c3", "grid:3x4", 3),
    ("grid2x3_def", "grid:2x3", None),
    ("grid1x2_def", "grid:1x2", None),
    ("grid2x2_def", "grid:2x2", None),
    ("grid4x5_def", "grid:4x5", None),
    ("grid3x3_c1", "grid:3x3", 1),
    ("grid7x7_slice", None, "grid_7x7_slice.txt"),
    ("b70_slice", None, "bristlecone_70_slice.txt"),
]


def bitstrings(seed, n, count):
    rng = np.random.Generator(np.random.PCG64(seed))
    return [format(int(v), f"0{n}b") for v in rng.integers(0, 2 ** n, size=count)]


def sab_draws(seed, n, count):
    rng = np.random.Generator(np.random.PCG64(seed))
    return ["".join(str(int(b)) for b in rng.integers(0, 2, size=n)) for _ in range(count)]


def cplx(v):
    return [float(np.real(v)), float(np.imag(v))]


def main():
    t0 = time.time()
    circ_obj, circ_text = {}, {}
    for key, lat, depth, seed, g in CIRCUITS:
        c = generate_rqc(Lattice.named(lat), depth, seed, two_qubit_gate=g)
        circ_obj[key] = c
        circ_text[key] = write_circuit(c)

    plan_obj, plan_text = {}, {}
    for key, lat, arg in GRID_PLANS:
        if lat is None:
            p = parse_plan(open(os.path.join(PLANS, arg)).read())
        elif arg is None:
            p = builtin_plan(Lattice.named(lat))
        else:
            p = grid_plan(Lattice.named(lat), n_cuts=arg)
        plan_obj[key] = p
        plan_text[key] = format_plan(p)

    amp_cases = []

    def amp_case(name, ckey, pkey, dtype, outs, in_bits=0, f=1.0, fseed=0):
        c = circ_obj[ckey]
        eng = AmplitudeEngine(c, plan_obj[pkey], dtype=dtype)
        fid = FidelitySpec(f=f, seed=fseed)
        amps, stats = [], None
        for o in outs:
            a, stats = eng.amplitude(in_bits, o, fid)
            amps.append(cplx(a))
        amp_cases.append({
            "name": name, "circuit": ckey, "plan": pkey,
            "dtype": np.dtype(dtype).name, "in_bits": in_bits if isinstance(in_bits, str)
            else format(in_bits, f"0{c.n}b"),
            "out_bits": outs, "f": f, "fseed": fseed, "amps": amps,
            "paths_total": stats.paths_total, "paths_used": stats.paths_used,
            "flops": stats.flops,
        })
        print(f"  amp {name}: {len(outs)} amps, {time.time() - t0:.1f}s", flush=True)

    amp_case("config1_c64", "g4x4_t16_s0", "grid4x4_c0", np.complex64, bitstrings(0, 16, 64))
    amp_case("config1_c128", "g4x4_t16_s0", "grid4x4_c0", np.complex128, bitstrings(0, 16, 8))
    amp_case("config2_c64", "g5x5_t24_s0", "grid5x5_c1", np.complex64, bitstrings(0, 25, 48))
    amp_case("g4x4s3_cuts2_f05", "g4x4_t16_s3", "grid4x4_c2", np.complex128,
             bitstrings(1, 16, 8), f=0.5, fseed=1)
    amp_case("g4x4s3_cuts2_f025_c64", "g4x4_t16_s3", "grid4x4_c2", np.complex64,
             bitstrings(2, 16, 8), f=0.25, fseed=7)
    amp_case("g4x4s3_in_nonzero", "g4x4_t16_s3", "grid4x4_def", np.complex128, [format(99, "016b")],
             in_bits="0000111100001111")
    amp_case("g3x4_cuts3", "g3x4_t12_s8", "grid3x4_c3", np.complex128, bitstrings(3, 12, 4))
    amp_case("g3x4_cuts1_c64", "g3x4_t16_s11", "grid3x4_c1", np.complex64, bitstrings(4, 12, 8))
    amp_case("g2x3_iswap", "g2x3_t10_s5_iswap", "grid2x3_def", np.complex128, bitstrings(5, 6, 8))
    amp_case("g1x2", "g1x2_t8_s1", "grid1x2_def", np.complex128, bitstrings(6, 2, 4))
    amp_case("g2x2", "g2x2_t9_s2", "grid2x2_def", np.complex64, bitstrings(7, 4, 4))
    amp_case("g3x3_depth0", "g3x3_t0_s4", "grid3x3_c1", np.complex128, bitstrings(8, 9, 4))
    amp_case("g4x5_def_c64", "g4x5_t24_s7", "grid4x5_def", np.complex64, bitstrings(9, 20, 4))
    amp_case("g7x7_t16_slice_f1", "g7x7_t16_s0", "grid7x7_slice", np.complex64, bitstrings(0, 49, 3))
    amp_case("g7x7_t16_slice_f64", "g7x7_t16_s0", "grid7x7_slice", np.complex64,
             bitstrings(10, 49, 3), f=1 / 64, fseed=0)
    amp_case("g7x7_t24_slice_f64", "g7x7_t24_s0", "grid7x7_slice", np.complex64,
             bitstrings(13, 49, 2), f=1 / 64, fseed=0)
    amp_case("b70_t8_slice_f1", "b70_t8_s0", "b70_slice", np.complex64, sab_draws(11, 70, 2))

    batch_cases = []

    def batch_case(name, ckey, pkey, dtype, s_ab, c_sites, n_c, seed, f=1.0, fseed=0, in_bits=0):
        c = circ_obj[ckey]
        eng = AmplitudeEngine(c, plan_obj[pkey], dtype=dtype)
        b = eng.amplitude_batch(in_bits, s_ab, c_sites, n_c, seed=seed,
                                fidelity=FidelitySpec(f=f, seed=fseed))
        batch_cases.append({
            "name": name, "circuit": ckey, "plan": pkey, "dtype": np.dtype(dtype).name,
            "in_bits": format(in_bits, f"0{c.n}b"), "s_ab": b.s_ab, "c_sites": list(c_sites),
            "n_c": n_c, "seed": seed, "f": f, "fseed": fseed,
            "c_values": list(b.c_values), "amps": [cplx(a) for a in b.amplitudes],
            "out_bits": [b.out_bits(i) for i in range(len(b))],
            "paths_used": b.stats.paths_used, "paths_total": b.stats.paths_total,
            "flops": b.stats.flops,
        })
        print(f"  batch {name}: {time.time() - t0:.1f}s", flush=True)

    batch_case("g4x4s3_b32", "g4x4_t16_s3", "grid4x4_def", np.complex128,
               "11110000" + "0" * 8, tuple(range(8, 16)), 32, 5)
    batch_case("g4x4s3_b16full", "g4x4_t16_s3", "grid4x4_def", np.complex128,
               "0" * 16, (12, 13, 14, 15), 16, 0)
    batch_case("g4x4s3_b8_c64", "g4x4_t16_s3", "grid4x4_c2", np.complex64,
               "1010101001010000", (12, 13, 14, 15), 8, 2, f=0.5, fseed=3)
    s_ab = sab_draws(12, 70, 3)
    batch_case("b70_t8_b64_f1", "b70_t8_s0", "b70_slice", np.complex64, s_ab[0],
               (8, 15, 16, 24, 25, 26), 64, 0)
    batch_case("b70_t16_b64_f64", "b70_t16_s0", "b70_slice", np.complex64, s_ab[1],
               (8, 15, 16, 24, 25, 26), 64, 0, f=1 / 64, fseed=0)
    batch_case("b70_t16_b64_f0005", "b70_t16_s0", "b70_slice", np.complex64, s_ab[2],
               (8, 15, 16, 24, 25, 26), 64, 0, f=0.005, fseed=0)

    batch_case("b70_t24_b64_f0005", "b70_t24_s0", "b70_slice", np.complex64, sab_draws(14, 70, 1)[0],
               (8, 15, 16, 24, 25, 26), 64, 0, f=0.005, fseed=0)

    costs = {}
    for pkey, ckey, opn in [("grid7x7_slice", "g7x7_t40_s0", ()),
                            ("b70_slice", "b70_t32_s0", (8, 15, 16, 24, 25, 26)),
                            ("grid5x5_c1", "g5x5_t24_s0", ()),
                            ("grid4x4_c0", "g4x4_t16_s0", ()),
                            ("grid7x7_slice", "g7x7_t16_s0", ()),
                            ("b70_slice", "b70_t16_s0", (8, 15, 16, 24, 25, 26)),
                            ("grid7x7_slice", "g7x7_t24_s0", ()),
                            ("b70_slice", "b70_t24_s0", (8, 15, 16, 24, 25, 26))]:
        c = circ_obj[ckey]
        e = estimate_cost(plan_obj[pkey], c.lattice, c.depth, open_sites=opn)
        costs[f"{pkey}@{ckey}"] = {
            "paths": e.paths, "total_flops": e.total_flops, "peak_bytes": e.peak_bytes,
            "open_sites": list(opn),
            "steps": [[s.name, s.flops, s.out_entries, s.evaluations] for s in e.steps],
        }

    out = {"generator": "tests/golden/make_golden.py (reference rqcsim 0.1.0)",
           "numpy": np.__version__,
           "circuits": circ_text, "plans": plan_text,
           "amplitudes": amp_cases, "batches": batch_cases, "costs": costs}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)

    # permutations: reference permute_fast (L/R move kernels) bytes, hashed
    rng = np.random.default_rng(91)
    perm_cases = []
    for i in range(60):
        rank = int(rng.integers(1, 9))
        while True:
            dims = [int(rng.integers(1, 5)) for _ in range(rank)]
            if math.prod(dims) <= 1 << 16:
                break
        perm = [int(p) for p in rng.permutation(rank)]
        perm_cases.append((dims, perm))
    for rank in (10, 12, 14, 16, 18):
        perm_cases.append(([2] * rank, [int(p) for p in rng.permutation(rank)]))
    for dims in ([4, 2, 8, 16, 2, 4, 2, 8], [16, 16, 8, 4, 2, 2, 4], [3, 5, 7, 2, 4],
                 [1, 1, 2, 1, 3], [32, 32, 32], [1]):
        perm_cases.append((dims, [int(p) for p in rng.permutation(len(dims))]))
    perm_cases.append(([2] * 7, [2, 5, 4, 0, 3, 6, 1]))   # worked example abcdefg->cfeadgb
    perms = []
    for j, (dims, perm) in enumerate(perm_cases):
        g = np.random.default_rng(1000 + j)
        x = (g.standard_normal(dims) + 1j * g.standard_normal(dims)).astype(np.complex64)
        fast = permute_fast(x, plan_permutation(dims, perm))
        naive = permute_naive(x, perm)
        assert fast.tobytes() == naive.tobytes()
        perms.append({"dims": dims, "perm": perm, "input_seed": 1000 + j,
                      "sha256": hashlib.sha256(np.ascontiguousarray(fast).tobytes()).hexdigest()})
    with open(os.path.join(HERE, "golden_perm.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py (reference permute_fast)",
                   "input": "np.random.default_rng(input_seed): (standard_normal(dims) + "
                            "1j*standard_normal(dims)).astype(complex64)",
                   "cases": perms}, fh, indent=1)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
