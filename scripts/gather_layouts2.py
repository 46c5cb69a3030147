"""Shapes + offset-table heads of the gathered GEMMs of one config-2 step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import tensor_core as tc
orig = tc.gemm_gather_buffer
seen = set()
def spy(batch, M, N, K, A, sA, roff, coff, B, opB, C, mode=None):
    key = (M, N, K, opB, tuple(roff[:4].tolist()), tuple(coff[:12].tolist()))
    if key not in seen:
        seen.add(key)
        print(f"M={M} N={N} K={K} opB={opB} roff[:4]={roff[:4].tolist()} coff[:12]={coff[:12].tolist()}")
    return orig(batch, M, N, K, A, sA, roff, coff, B, opB, C, mode)
tc.gemm_gather_buffer = spy
lat = qf.Lattice.named("grid:5x5"); circ = qf.generate_rqc(lat, "1+24+1", 0)
eng = qf.AmplitudeEngine(circ, qf.grid_plan(lat, n_cuts=1))
rng = np.random.Generator(np.random.PCG64(0))
outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=1024)]
eng.amplitudes(0, outs)
