"""Diagnose TMA-fed tensor-core GEMM against float64 for small-N shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1811_09599_b200 import _lib, tensor_core as tc
lib = _lib.load()
rng = np.random.default_rng(0)
for var in (20,):
    lib.qf_tc3_set_variant(var)
    for (b, M, N, K, ob) in [(64, 512, 8, 64, 0), (64, 512, 64, 64, 0), (64, 512, 16, 64, 0), (64, 512, 32, 64, 0),
                             (64, 512, 48, 64, 0), (256, 512, 64, 64, 0), (64, 512, 8, 32, 0), (64, 512, 8, 128, 0)]:
        A = (rng.standard_normal((b, M, K)) + 1j * rng.standard_normal((b, M, K))).astype(np.complex64)
        B = (rng.standard_normal((b, K, N) if ob == 0 else (b, N, K)) + 0j).astype(np.complex64)
        C = torch.zeros(b * M * N, dtype=torch.complex64, device="cuda")
        tc.gemm_buffer(b, M, N, K, torch.from_numpy(A.reshape(-1)).cuda(), 0,
                       torch.from_numpy(B.reshape(-1)).cuda(), ob, C, mode=2)
        Bm = B if ob == 0 else B.transpose(0, 2, 1)
        want = np.matmul(A.astype(np.complex128), Bm.astype(np.complex128))
        got = C.cpu().numpy().reshape(b, M, N)
        err = np.abs(got - want)
        bad = np.argwhere(err > 1e-3 * np.abs(want).max())
        print(var, (b, M, N, K, ob), "rel", float(np.linalg.norm(got - want) / np.linalg.norm(want)),
              "bad", len(bad), bad[:4].tolist())
