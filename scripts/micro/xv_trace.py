"""Trace expand_plan decisions in one config-2 call (which operand pairs fuse)."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import tensor_core as tc, contraction_plan as cp
orig = cp.expand_plan
def traced(acc, op, op2, late, tail2=()):
    r = orig(acc, op, op2, late, tail2)
    print("PAIR", list(zip(acc.labels, acc.dims))[:12], "|", op.labels, "|", op2.labels, "->",
          None if r is None else (r["M"], r["K"], r["N"], r.get("open"), r.get("view") is not None))
    return r
cp.expand_plan = traced
lat = qf.Lattice.named("grid:5x5"); circ = qf.generate_rqc(lat, "1+24+1", 0)
eng = qf.AmplitudeEngine(circ, qf.grid_plan(lat, n_cuts=1))
rng = np.random.Generator(np.random.PCG64(0))
outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=1024)]
eng.amplitudes(0, outs)
