"""N = 8 / 16 GEMM shapes of the config-2 step under every engine."""
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

lib = _lib.load()
for (b, M, N, K, oa, ob) in [(1024, 4096, 8, 64, 0, 0), (1024, 4096, 8, 64, 1, 0), (1024, 4096, 16, 64, 0, 0),
                             (1024, 4096, 8, 32, 0, 0), (2, 8388608, 8, 8, 0, 0), (1024, 32768, 8, 8, 0, 0)]:
    A = torch.randn(b * M * K, dtype=torch.complex64, device="cuda")
    B = torch.randn(b * K * N, dtype=torch.complex64, device="cuda")
    C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
    byts = 8 * b * (M * K + K * N + M * N)
    row = {}
    for name, mode, eng, var in (("auto", 0, 0, 0), ("smem", 1, 1, 0), ("rowblock", 1, 2, 0), ("rowstream", 1, 3, 0),
                                 ("tc3", 2, 0, 0), ("tc3_8w", 2, 0, 10), ("tc3_16w", 2, 0, 11)):
        lib.qf_small_engine(eng); lib.qf_tc3_set_variant(var)
        try:
            ms = timeit(lambda: tc.gemm_buffer(b, M, N, K, A, oa, B, ob, C, mode=mode), 5)
            row[name] = f"{ms:.3f}ms {byts / ms / 1e6:.0f}GB/s"
        except Exception as e:
            row[name] = f"err {str(e)[:40]}"
    lib.qf_small_engine(0); lib.qf_tc3_set_variant(0)
    print(f"{b}x({M},{N},{K}) op{oa}{ob}: {row}", flush=True)
