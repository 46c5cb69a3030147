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
alpha = 0.5
C = torch.zeros(b * M * N, dtype=torch.complex64, device="cuda")
tc.gemm_buffer(b, M, N, K, torch.from_numpy(A.reshape(-1)).cuda(), 0, torch.from_numpy(B.reshape(-1)).cuda(), 0, C, alpha, 0.0, mode=2)
want = alpha * np.matmul(A.astype(np.complex128), B.astype(np.complex128))
got = C.cpu().numpy().reshape(b, M, N)
g_ = got[0, 128:256]; w_ = want[0, 128:256]
bad = np.abs(g_ - w_) > 1e-4 * np.abs(w_).max()
print("bad rows", np.nonzero(bad.any(1))[0].tolist()[:64])
print("bad cols", np.nonzero(bad.any(0))[0].tolist())
r = np.nonzero(bad.any(1))[0][0]
print("row", r, "got", g_[r, :4], "want", w_[r, :4], "ratio", (g_[r, :4] / w_[r, :4]))
