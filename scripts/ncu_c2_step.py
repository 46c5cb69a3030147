"""One config-2 amplitudes() call (1024 bit-strings, late output slicing)
between cudaProfilerStart/Stop, after two warm-up calls -- for
`ncu --profile-from-start off` captures of exactly one step."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_09599_b200 as qf
lat = qf.Lattice.named("grid:5x5"); circ = qf.generate_rqc(lat, "1+24+1", 0)
eng = qf.AmplitudeEngine(circ, qf.grid_plan(lat, n_cuts=1))
rng = np.random.Generator(np.random.PCG64(0))
outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=1024)]
for _ in range(2):
    eng.amplitudes(0, outs, graph=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
eng.amplitudes(0, outs, graph=True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
