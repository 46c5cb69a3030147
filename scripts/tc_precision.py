"""Diagnostic: relative error of the complex GEMM engines vs float64, by K."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1811_09599_b200 import _lib, tensor_core as tc

def err(M, N, K, mode, variant=0, seed=0, scale_lo=False):
    rng = np.random.default_rng(seed)
    A = (rng.standard_normal((M, K)) + 1j * rng.standard_normal((M, K))).astype(np.complex64)
    B = (rng.standard_normal((K, N)) + 1j * rng.standard_normal((K, N))).astype(np.complex64)
    lib = _lib.load(); lib.qf_tc3_set_variant(variant)
    C = torch.empty(M * N, dtype=torch.complex64, device="cuda")
    tc.gemm_buffer(1, M, N, K, torch.from_numpy(A.reshape(-1)).cuda(), 0,
                   torch.from_numpy(B.reshape(-1)).cuda(), 0, C, mode=mode)
    got = C.cpu().numpy().reshape(M, N)
    want = A.astype(np.complex128) @ B.astype(np.complex128)
    return np.linalg.norm(got - want) / np.linalg.norm(want), np.max(np.abs(got - want) / np.abs(want).mean())

for K in (8, 16, 64, 256, 1000, 4096, 32768):
    r = [err(256, 128, K, m, v) for m, v in ((1, 0), (2, 1), (2, 0))]
    print(f"K={K:5d}  ffma {r[0][0]:.2e}  tc-v1 {r[1][0]:.2e}  tc-promoted {r[2][0]:.2e}   (max {r[0][1]:.1e} {r[1][1]:.1e} {r[2][1]:.1e})")
