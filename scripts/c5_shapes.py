"""Config-5 GEMM shapes across tensor-core kernel flavours (TFLOP/s)."""
import sys, os
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
lib = _lib.load()
for (b, M, N, K, oa, ob) in [(1, 1048576, 256, 256, 0, 0), (1, 1048576, 256, 256, 0, 1), (1, 4194304, 256, 256, 0, 0),
                             (1, 2097152, 512, 256, 0, 0), (1, 65536, 256, 256, 0, 0), (1, 4096, 4096, 65536, 0, 0),
                             (1, 1048576, 256, 16, 0, 0), (1, 16777216, 32, 16, 0, 0)]:
    A = torch.randn(b * M * K, dtype=torch.complex64, device="cuda")
    B = torch.randn(b * K * N, dtype=torch.complex64, device="cuda")
    C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
    row = {}
    for name, var in (("auto", 0), ("8w", 10), ("16w", 11), ("16w+epi", 12), ("long-ck4", 13), ("long-ck8", 14)):
        lib.qf_tc3_set_variant(var)
        try:
            ms = timeit(lambda: tc.gemm_buffer(b, M, N, K, A, oa, B, ob, C, mode=2))
            row[name] = round(8 * b * M * N * K / ms / 1e9, 1)
        except Exception as e:
            row[name] = "err"
    lib.qf_tc3_set_variant(0)
    print(f"{b}x({M},{N},{K}) op{oa}{ob} TFLOP/s: {row}", flush=True)
