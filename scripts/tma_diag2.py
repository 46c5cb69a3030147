import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1811_09599_b200 import _lib, tensor_core as tc
lib = _lib.load()
rng = np.random.default_rng(0)
for var in (10, 11, 12, 17, 20):
  lib.qf_tc3_set_variant(var)
  for (b, M, N, K, ob) in [(64, 512, 64, 64, 0)]:
    for alpha, beta in ((0.5, 0.0), (1.0, 0.5)):
        A = (rng.standard_normal((b, M, K)) + 1j * rng.standard_normal((b, M, K))).astype(np.complex64)
        B = (rng.standard_normal((b, K, N)) + 0j).astype(np.complex64)
        C0 = (rng.standard_normal((b, M, N)) + 0j).astype(np.complex64)
        C = torch.from_numpy(C0.reshape(-1)).cuda()
        tc.gemm_buffer(b, M, N, K, torch.from_numpy(A.reshape(-1)).cuda(), 0,
                       torch.from_numpy(B.reshape(-1)).cuda(), ob, C, alpha, beta, mode=2)
        want = alpha * np.matmul(A.astype(np.complex128), B.astype(np.complex128)) + beta * C0
        got = C.cpu().numpy().reshape(b, M, N)
        print(var, (b, M, N, K), alpha, beta, "rel", float(np.linalg.norm(got - want) / np.linalg.norm(want)))
