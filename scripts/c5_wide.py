"""Config-4/5 GEMM shapes: the 64-column Gauss kernel (variant 32 / the K <= 256
path) against the wide kernel, single CTAs (40) and CTA pairs (43).
QF_TC3W_MINK=256 lets the wide kernel take the K = 256 shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1811_09599_b200 import _lib, tensor_core as tc
def timeit(fn, reps=8):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
lib = _lib.load()
for (b, M, N, K, oa, ob) in [(1, 1048576, 256, 256, 0, 0), (1, 1048576, 256, 256, 0, 1), (1, 4194304, 256, 256, 0, 0),
                             (1, 2097152, 512, 256, 0, 0), (1, 65536, 256, 256, 0, 0), (1, 32768, 1024, 1024, 0, 0),
                             (1, 1048576, 1024, 1024, 0, 1), (1, 32768, 32768, 1024, 0, 0), (1, 4096, 4096, 512, 0, 0)]:
    A = torch.randn(b * M * K, dtype=torch.complex64, device="cuda")
    B = torch.randn(b * K * N, dtype=torch.complex64, device="cuda")
    C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
    row = {}
    for name, var in (("narrow", 32), ("wide", 40), ("pair", 43), ("pair-ck128", 44), ("auto", 0)):
        lib.qf_tc3_set_variant(var)
        try:
            ms = timeit(lambda: tc.gemm_buffer(b, M, N, K, A, oa, B, ob, C, mode=2))
            row[name] = (round(8 * b * M * N * K / ms / 1e9, 1), _lib.last_kernel())
        except Exception as e:
            row[name] = "err " + str(e)[:60]
    lib.qf_tc3_set_variant(0)
    print(f"{b}x({M},{N},{K}) op{oa}{ob} TFLOP/s: {row}", flush=True)
