"""Trace PlanExecutor._defer decisions in one config-2 call."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import tensor_core as tc, contraction_plan as cp
orig_defer = cp.PlanExecutor._defer
def traced(self, step, path, values, acc, op):
    users = [s for s in self.plan.steps() if step.name in s.inputs]
    print("DEFER?", step.name, [u.name for u in users], [u.inputs for u in users][:2], acc.labels[:3], op.labels)
    r = orig_defer(self, step, path, values, acc, op)
    print("  ->", r is not None)
    return r
cp.PlanExecutor._defer = traced
orig = cp.expand_plan
def traced2(acc, op, op2, late, tail2=()):
    r = orig(acc, op, op2, late, tail2)
    print("  PLAN", acc.labels, op.labels, op2.labels, tail2, "->", None if r is None else (r["M"], r["K"], r["N"]))
    return r
cp.expand_plan = traced2
lat = qf.Lattice.named("grid:5x5"); circ = qf.generate_rqc(lat, "1+24+1", 0)
eng = qf.AmplitudeEngine(circ, qf.grid_plan(lat, n_cuts=1))
rng = np.random.Generator(np.random.PCG64(0))
outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=1024)]
eng.amplitudes(0, outs)
