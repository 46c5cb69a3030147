"""Per-case permutation GB/s for config 3 (CUDA-graph timing), with the
planner's tile decision (QF_PERM_DEBUG), to find the slowest shapes.
Usage: QF_PERM_DEBUG=1 python scripts/perm_cases.py 28 > out.txt"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import config3_cases  # noqa: E402
from paper_1811_09599_b200 import tensor_core as tc  # noqa: E402

log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
steps = 10
n = 1 << log2n
src = torch.randn(n, dtype=torch.complex64, device="cuda")
dst = torch.empty_like(src)
res = []
for i, (dims, perm) in enumerate(config3_cases(log2n, 64, seed=log2n)):
    for _ in range(3):
        tc.permute_buffer(src, dims, perm, out=dst)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
        for _ in range(steps):
            tc.permute_buffer(src, dims, perm, out=dst)
    torch.cuda.current_stream().wait_stream(cs)
    g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    gbs = 16 * n / (a.elapsed_time(b) / steps) / 1e6
    res.append((gbs, i, dims, perm))
    print(f"case {i} {gbs:.1f} GB/s dims {dims} perm {perm}", flush=True)
res.sort()
print("slowest:")
for r in res[:8]:
    print(f"  {r[0]:.1f} case {r[1]} dims {r[2]} perm {r[3]}")
print(f"mean {np.mean([r[0] for r in res]):.1f}")
