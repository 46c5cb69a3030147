"""Run one labelled contraction a few times (ncu target).
usage: contract_one.py '<a labels>' '<b labels>' dim reps   (labels space-separated, batch '@b' 1024)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_09599_b200 import tensor_core as tc
al, bl, dim, reps = sys.argv[1].split(), sys.argv[2].split(), int(sys.argv[3]), int(sys.argv[4])
if len(sys.argv) > 5:  # K3 small-engine override (0 auto, 2 row-block, 3 row-stream)
    from paper_1811_09599_b200 import _lib
    _lib.load().qf_small_engine(int(sys.argv[5]))
shape = lambda ls: tuple(1024 if l == "@b" else dim for l in ls)
a = tc.Tensor(al, torch.randn(shape(al), dtype=torch.complex64, device="cuda").reshape(-1), shape(al))
b = tc.Tensor(bl, torch.randn(shape(bl), dtype=torch.complex64, device="cuda").reshape(-1), shape(bl))
for _ in range(reps):
    tc.contract(a, b)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(10): tc.contract(a, b)
ev[1].record(); torch.cuda.synchronize()
print("ms", ev[0].elapsed_time(ev[1]) / 10)
