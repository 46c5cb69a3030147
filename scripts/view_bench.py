"""Dominant config-2 GEMM shape 1024 x (4096 x 64 x 64): plain N (TMA), the
5-D TMA view, offset tables; and ring/converter variants."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
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
B = torch.randn(nb * K * N, dtype=torch.complex64, device="cuda")
C = torch.empty(nb * M * N, dtype=torch.complex64, device="cuda")
lib = _lib.load()
def rep(name, ms): print(f"{name:40s} {ms:.3f} ms {byts / ms / 1e6:.0f} GB/s", flush=True)
for var in (21, 22):
    lib.qf_tc3_set_variant(var)
    rep(f"plain NN variant {var}", timeit(lambda: tc.gemm_buffer(nb, M, N, K, A, 0, B, 0, C)))
    ta = tc.Tensor(("@b", "p", "s", "q", "r", "x", "t"), A, (nb, 8, 8, 8, 8, 8, 8))
    tb = tc.Tensor(("@b", "s", "t", "v", "w"), B, (nb, 8, 8, 8, 8))
    rep(f"view variant {var}", timeit(lambda: tc.contract(ta, tb)))
lib.qf_tc3_set_variant(0)
rep("plain NN (auto)", timeit(lambda: tc.gemm_buffer(nb, M, N, K, A, 0, B, 0, C)))
# view: A entry [p(8) s(8) q(8) r(8) t(8) x(8)] as rows (p, q, r, x?) ... labels
dims = (8, 8, 8, 8, 8, 8)
for lab, desc in ((("p", "s", "q", "r", "x", "t"), "view kout mid"),
                  (("p", "q", "r", "s", "x", "t"), "view kout late"),
                  (("s", "p", "q", "r", "x", "t"), "view kout first")):
    ta = tc.Tensor(("@b",) + lab, A, (nb,) + dims)
    tb = tc.Tensor(("@b", "s", "t", "v", "w"), B, (nb, 8, 8, 8, 8))
    rep(desc, timeit(lambda: tc.contract(ta, tb)))
    prev = tc.set_view(False)
    rep(desc + " (tables)", timeit(lambda: tc.contract(ta, tb)))
    tc.set_view(prev)
