import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1811_09599_b200 import tensor_core as tc, _lib
rng = np.random.default_rng(0)
nb = 4
A = (rng.standard_normal((nb, 8, 8, 16, 8, 8)) + 0j).astype(np.complex64)
S = (rng.standard_normal((8, 8, 8, 8, 2)) + 0j).astype(np.complex64)
W = (rng.standard_normal((8, 8, 8, 8, 2)) + 0j).astype(np.complex64)
bits = rng.integers(0, 2, size=(2, nb)).astype(np.int32)
late = tc.LateBits(torch.from_numpy(bits).cuda(), {"out0": 0, "out1": 1})
ta = tc.Tensor(["@b", "r", "p", "q", "j1", "j2"], A)
ts = tc.Tensor(["j1", "j2", "t", "u", "out0"], S)
tw = tc.Tensor(["r", "u", "v", "w", "out1"], W)
plan = tc.expand_plan(ta, ts, tw, late)
print({k: v for k, v in plan.items() if k not in ("u",)})
r = tc.contract_late_expand(ta, ts, tw, late, plan)
print("result", r is not None, _lib.load().qf_last_error())
