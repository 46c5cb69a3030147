import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1811_09599_b200 import _lib, tensor_core as tc
lib = _lib.load()
rng = np.random.default_rng(0)
b, M, N, K = 16, 1024, 128, 512
A = (rng.standard_normal((b, M, K)) + 1j * rng.standard_normal((b, M, K))).astype(np.complex64)
B = (rng.standard_normal((b, K, N)) + 0j).astype(np.complex64)
dA, dB = torch.from_numpy(A.reshape(-1)).cuda(), torch.from_numpy(B.reshape(-1)).cuda()
want1 = np.matmul(A.astype(np.complex128), B.astype(np.complex128))
for var in (13, 19):
    lib.qf_tc3_set_variant(var)
    for alpha in (1.0, 0.5, 0.5 - 1j):
        C = torch.zeros(b * M * N, dtype=torch.complex64, device="cuda")
        tc.gemm_buffer(b, M, N, K, dA, 0, dB, 0, C, alpha, 0.0, mode=2)
        got = C.cpu().numpy().reshape(b, M, N); want = alpha * want1
        errs = [float(np.linalg.norm(got[i] - want[i]) / np.linalg.norm(want[i])) for i in range(b)]
        tiles_bad = [(i, t) for i in range(b) for t in range(16) if np.linalg.norm(got[i, (t//2)*128:(t//2+1)*128, (t%2)*64:(t%2+1)*64] - want[i, (t//2)*128:(t//2+1)*128, (t%2)*64:(t%2+1)*64]) > 1e-4 * np.linalg.norm(want[i, (t//2)*128:(t//2+1)*128, (t%2)*64:(t%2+1)*64])]
        print(var, alpha, "max batch err", f"{max(errs):.2e}", "bad tiles", len(tiles_bad), [i*16+t for i, t in tiles_bad][:12])
