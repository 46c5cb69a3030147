"""Per-case config-3 permutation timings (CUDA events), optional case filter:
python scripts/perm_one.py LOG2N [first] [count]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1811_09599_b200 import tensor_core as tc
log2n = int(sys.argv[1]); first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 64
n = 1 << log2n
src = torch.randn(n, dtype=torch.complex64, device="cuda"); dst = torch.empty_like(src)
cases = bench.config3_cases(log2n, 64, seed=log2n)
for i in range(first, min(64, first + count)):
    dims, perm = cases[i]
    for _ in range(3): tc.permute_buffer(src, dims, perm, out=dst)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): tc.permute_buffer(src, dims, perm, out=dst)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"case {i:2d} {16 * n / ms / 1e6:7.0f} GB/s  dims {dims} perm {perm}", flush=True)
