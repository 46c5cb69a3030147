"""A/B one GEMM shape across engines: python shape_ab.py b M N K [opA opB]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_09599_b200 import _lib, tensor_core as tc
b, M, N, K = (int(x) for x in sys.argv[1:5])
oa, ob = (int(sys.argv[5]), int(sys.argv[6])) if len(sys.argv) > 6 else (0, 0)
def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return a.elapsed_time(e) / reps
A = torch.randn(b * M * K, dtype=torch.complex64, device="cuda")
B = torch.randn(b * K * N, dtype=torch.complex64, device="cuda")
C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
byts = 8 * b * (M * K + K * N + M * N)
for name, mode in (("simt", 1), ("tc3", 2), ("auto", 0)):
    ms = timeit(lambda: tc.gemm_buffer(b, M, N, K, A, oa, B, ob, C, mode=mode))
    print(f"{b}x({M},{N},{K}) op{oa}{ob} {name}: {ms:.3f} ms {byts / ms / 1e6:.0f} GB/s")
