"""Drop-in single-call rate: AmplitudeEngine.amplitude (one bit-string per
call, rq/amplitude_engine.py:114-126) on config 2, host wall time per call,
plus a cProfile of the host side of one call."""
import cProfile
import json
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1811_09599_b200 as qf

lat = qf.Lattice.named("grid:5x5")
circ = qf.generate_rqc(lat, "1+24+1", 0)
plan = qf.grid_plan(lat, n_cuts=1)
eng = qf.AmplitudeEngine(circ, plan)
rng = np.random.Generator(np.random.PCG64(0))
outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=64)]
for o in outs[:4]:
    eng.amplitude(0, o)
torch.cuda.synchronize()
t0 = time.perf_counter()
for o in outs:
    eng.amplitude(0, o)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / len(outs)
pr = cProfile.Profile()
pr.enable()
for o in outs[:8]:
    eng.amplitude(0, o)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(25)
print(json.dumps({"single_call_ms": round(dt * 1e3, 3), "amp_per_s": round(1 / dt, 1)}))
