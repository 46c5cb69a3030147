"""Time the slowest config-3 shapes (disjoint 64 x 64 tiles) under planner
knobs given in the environment (QF_PERM_TA / QF_PERM_TB / QF_PERM_TILE)."""
import sys

import torch

sys.path.insert(0, ".")
from bench import config3_cases  # noqa: E402
from paper_1811_09599_b200 import tensor_core as tc  # noqa: E402

picks = {28: [35, 58, 32, 56, 50, 34, 0, 16], 24: [56, 9, 17, 38, 60]}
tot = []
for log2n, ids in picks.items():
    n = 1 << log2n
    src = torch.randn(n, dtype=torch.complex64, device="cuda")
    dst = torch.empty_like(src)
    cases = config3_cases(log2n, 64, seed=log2n)
    for i in ids:
        dims, perm = cases[i]
        for _ in range(3):
            tc.permute_buffer(src, dims, perm, out=dst)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
            for _ in range(10):
                tc.permute_buffer(src, dims, perm, out=dst)
        torch.cuda.current_stream().wait_stream(cs)
        g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ref = src.view(dims).permute(perm).contiguous().view(-1)
        ok = torch.equal(ref, dst)
        gbs = 16 * n / (a.elapsed_time(b) / 10) / 1e6
        tot.append(gbs)
        print(f"2^{log2n} case {i} {gbs:.1f} GB/s exact={ok}", flush=True)
    del src, dst
print(f"mean {sum(tot) / len(tot):.1f}")
