"""Print operand layouts of every late-path contraction of one config-2 walk
and time the sliced (SN) GEMM under each CUDA-core engine."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import tensor_core as tc, _lib
lat = qf.Lattice.named("grid:5x5"); circ = qf.generate_rqc(lat, "1+24+1", 0)
eng = qf.AmplitudeEngine(circ, qf.grid_plan(lat, n_cuts=1))
rng = np.random.Generator(np.random.PCG64(0))
outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=1024)]
orig = tc.contract_late
def spy(a, b, late, tail=()):
    print("A", list(zip(a.labels, a.dims)), "\n B", list(zip(b.labels, b.dims)), flush=True)
    r = orig(a, b, late, tail)
    print(" ->", list(zip(r.labels, r.dims)), flush=True)
    return r
tc.contract_late = spy
import paper_1811_09599_b200.contraction_plan as cp
cp.contract_late = spy
eng.amplitudes(0, outs)
cp.contract_late = orig
lib = _lib.load()
for e in (0, 1, 2, 3):
    lib.qf_small_engine(e)
    for _ in range(2): eng.amplitudes(0, outs)
    with tc.KernelTimer() as kt:
        eng.amplitudes(0, outs)
    s = kt.summary(detail=True)
    print("engine", e, {k: round(d["ms"], 3) for k, d in s.items() if " S" in k or "n8 k64" in k})
lib.qf_small_engine(0)
