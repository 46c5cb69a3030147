"""GEMM engine throughput (algorithmic 8*M*N*K complex flops) + TF32 peak."""
import sys, os, json
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

def tf32_peak():
    torch.backends.cuda.matmul.allow_tf32 = True
    x = torch.randn(8192, 8192, device="cuda"); y = torch.randn(8192, 8192, device="cuda")
    ms = timeit(lambda: x @ y, 10)
    return 2 * 8192**3 / ms / 1e9

out = {"tf32_cublas_tflops": round(tf32_peak(), 1)}
lib = _lib.load()
for (b, M, N, K) in [(1, 4096, 4096, 4096), (1, 8192, 8192, 8192), (1, 32768, 512, 32768 // 4),
                     (1024, 4096, 64, 64), (64, 4096, 64, 512), (1, 16384, 16384, 2048)]:
    A = torch.randn(b * M * K, dtype=torch.complex64, device="cuda")
    B = torch.randn(b * K * N, dtype=torch.complex64, device="cuda")
    C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
    row = {}
    for name, mode, var in (("ffma", 1, 0), ("tc3_default", 2, 0), ("tc3w_regs", 2, 15), ("tmem_ck8", 2, 14), ("tma", 2, 19)):
        lib.qf_tc3_set_variant(var)
        ms = timeit(lambda: tc.gemm_buffer(b, M, N, K, A, 0, B, 0, C, mode=mode), 5)
        row[name] = round(8 * b * M * N * K / ms / 1e9, 1)
    lib.qf_tc3_set_variant(0)
    out[f"{b}x({M},{N},{K})"] = row
    print(f"{b}x({M},{N},{K}) TFLOP/s: {row}", flush=True)
print(json.dumps(out))
