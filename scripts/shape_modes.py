"""Time given GEMM shapes under each engine choice (auto / FFMA / tc3):
python scripts/shape_modes.py  -> config-5 narrow shapes by default."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_09599_b200 import _lib, tensor_core as tc

def timeit(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

shapes = [(1, 67108864, 16, 16, 0, 0), (1, 16777216, 16, 16, 0, 0), (1, 16777216, 16, 16, 0, 1),
          (2, 8388608, 8, 8, 0, 0), (1024, 4096, 8, 64, 0, 0), (1024, 4096, 16, 64, 0, 0),
          (1024, 4096, 64, 8, 0, 0)]
for (b, M, N, K, oa, ob) in shapes:
    A = torch.randn(b * M * K, dtype=torch.complex64, device="cuda")
    B = torch.randn(b * K * N, dtype=torch.complex64, device="cuda")
    C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
    byts = 8 * b * (M * K + K * N + M * N)
    row = {}
    for name, mode in (("auto", 0), ("ffma", 1), ("tc3", 2)):
        try:
            ms = timeit(lambda: tc.gemm_buffer(b, M, N, K, A, oa, B, ob, C, mode=mode))
            row[name] = f"{ms:.3f}ms {byts / ms / 1e6:.0f}GB/s [{_lib.load().qf_last_kernel().decode()}]"
        except Exception as e:
            row[name] = f"err {str(e)[:50]}"
    print(f"{b}x({M},{N},{K}) op{oa}{ob}: {row}", flush=True)
    del A, B, C
