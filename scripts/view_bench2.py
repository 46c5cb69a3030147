"""Direct qf_cgemm_c64_view timings on one buffer described several ways."""
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

nb, M, N, K = 1024, 4096, 64, 64
byts = 8 * nb * (M * K + K * N + M * N)
A = torch.randn(nb * M * K, dtype=torch.complex64, device="cuda")
B = tc.Tensor(("@b", "k", "n"), torch.randn(nb * K * N, dtype=torch.complex64, device="cuda"), (nb, K, N))
C = torch.empty(nb * M * N, dtype=torch.complex64, device="cuda")
lib = _lib.load()
views = {"plain-as-view kin64": (64, 4096, 64, 1, 64, 1, M * K),
         "plain kin8 kout8 adjacent": (8, 4096, 64, 8, 8, 1, M * K),
         "kout mid (p s q r x t)": (8, 512, 8, 8, 4096, 8, 32768),
         "kout first (s p q r x t)": (8, 4096, 8, 8, 32768, 1, M * K),
         "rows_a 64 (q s r x p t)": (8, 64, 8, 8, 512, 64, 4096)}
for var in (21, 22):
    lib.qf_tc3_set_variant(var)
    ms = timeit(lambda: tc.gemm_buffer(nb, M, N, K, A, 0, B.data, 0, C))
    print(f"var {var} plain NN: {ms:.3f} ms {byts / ms / 1e6:.0f} GB/s", flush=True)
    for name, v in views.items():
        ok = [True]
        def run():
            ok[0] = tc._gemm_view(nb, M, N, K, A.data_ptr(), M * K, v, B, N, K * N, 0, C)
        ms = timeit(run)
        print(f"var {var} {name:28s}: {ms:.3f} ms {byts / ms / 1e6:.0f} GB/s launched={ok[0]}", flush=True)
lib.qf_tc3_set_variant(0)
