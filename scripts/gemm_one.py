"""Run one complex GEMM shape a few times (target for ncu captures).
usage: gemm_one.py batch M N K mode variant reps"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_09599_b200 import _lib, tensor_core as tc
b, M, N, K, mode, var, reps = (int(x) for x in sys.argv[1:8])
lib = _lib.load(); lib.qf_tc3_set_variant(var)
A = torch.randn(b * M * K, dtype=torch.complex64, device="cuda")
B = torch.randn(b * K * N, dtype=torch.complex64, device="cuda")
C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
for _ in range(reps):
    tc.gemm_buffer(b, M, N, K, A, 0, B, 0, C, mode=mode)
torch.cuda.synchronize()
print("ok")
