import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1811_09599_b200 import _lib, tensor_core as tc
lib = _lib.load()
for shape in [(1, 256, 64, 8), (1, 256, 64, 64), (1, 300, 100, 77), (2, 1000, 130, 1000), (3, 4096, 64, 64), (1, 2048, 2048, 512)]:
    b, M, N, K = shape
    rng = np.random.default_rng(0)
    A = (rng.standard_normal((b, M, K)) + 1j * rng.standard_normal((b, M, K))).astype(np.complex64)
    B = (rng.standard_normal((b, K, N)) + 1j * rng.standard_normal((b, K, N))).astype(np.complex64)
    want = np.matmul(A.astype(np.complex128), B.astype(np.complex128))
    for var in (0, 6):
        lib.qf_tc3_set_variant(var)
        C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
        tc.gemm_buffer(b, M, N, K, torch.from_numpy(A.reshape(-1)).cuda(), 0, torch.from_numpy(B.reshape(-1)).cuda(), 0, C, mode=2)
        torch.cuda.synchronize()
        got = C.cpu().numpy().reshape(b, M, N)
        print(shape, "variant", var, "rel err %.2e" % (np.linalg.norm(got - want) / np.linalg.norm(want)), flush=True)
