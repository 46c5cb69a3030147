import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1811_09599_b200 import _lib, tensor_core as tc
lib = _lib.load()
rng = np.random.default_rng(0)
lib.qf_tc3_set_variant(20)
b, M, N, K = 64, 512, 64, 64
A = (rng.standard_normal((b, M, K)) + 1j * rng.standard_normal((b, M, K))).astype(np.complex64)
B = (rng.standard_normal((b, K, N)) + 0j).astype(np.complex64)
for alpha in (0.5, 1.0):
    C = torch.zeros(b * M * N, dtype=torch.complex64, device="cuda")
    tc.gemm_buffer(b, M, N, K, torch.from_numpy(A.reshape(-1)).cuda(), 0, torch.from_numpy(B.reshape(-1)).cuda(), 0, C, alpha, 0.0, mode=2)
    want = alpha * np.matmul(A.astype(np.complex128), B.astype(np.complex128))
    got = C.cpu().numpy().reshape(b, M, N)
    for bi in (0, 1, 63):
        for t in range(4):
            g_ = got[bi, t*128:(t+1)*128]; w_ = want[bi, t*128:(t+1)*128]
            e = np.linalg.norm(g_ - w_) / np.linalg.norm(w_)
            # does the tile match the product of another batch's B?
            alt = [float(np.linalg.norm(g_ - alpha * A[bi, t*128:(t+1)*128] @ B[bj]) / np.linalg.norm(w_)) for bj in range(max(0, bi-2), min(b, bi+3))]
            print(alpha, bi, t, f"{e:.3e}", "alt-batch errs", [f"{x:.1e}" for x in alt])
