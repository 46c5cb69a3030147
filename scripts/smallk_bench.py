"""Short-K GEMM shapes of the config-2 step: SIMT engines vs the short-K
tensor-core kernel (GB/s of A + B + C traffic and TFLOP/s)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_09599_b200 import _lib, tensor_core as tc

def timeit(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

for (b, M, N, K, oa, ob) in [(1024, 4096, 64, 8, 0, 0), (1024, 512, 512, 8, 1, 1), (1024, 512, 512, 8, 0, 0),
                             (1024, 4096, 64, 16, 0, 0), (1024, 4096, 32, 8, 0, 0), (1024, 4096, 64, 32, 0, 0),
                             (1024, 32768, 8, 8, 0, 0), (1024, 4096, 8, 64, 0, 0), (1024, 4096, 8, 64, 1, 0),
                             (1024, 4096, 16, 64, 0, 0), (1024, 4096, 32, 64, 0, 0), (1024, 32768, 8, 8, 1, 1)]:
    A = torch.randn(b * M * K, dtype=torch.complex64, device="cuda")
    B = torch.randn(b * K * N, dtype=torch.complex64, device="cuda")
    C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
    byts = 8 * b * (M * K + K * N + M * N)
    row = {}
    for name, mode, var in (("simt", 1, 0), ("tc3", 2, 0), ("tc3_8w", 2, 10), ("tc3_16w", 2, 11), ("tc3_epi", 2, 12), ("tc3_tma", 2, 20)):
        _lib.load().qf_tc3_set_variant(var)
        try:
            ms = timeit(lambda: tc.gemm_buffer(b, M, N, K, A, oa, B, ob, C, mode=mode), 5)
            row[name] = f"{ms:.3f} ms {byts / ms / 1e6:.0f} GB/s {8 * b * M * N * K / ms / 1e9:.1f} TF/s"
        except Exception as e:
            row[name] = f"err {e}"
    print(f"{b}x({M},{N},{K}) op{oa}{ob}: {row}", flush=True)
