"""HBM bandwidth by direction (torch kernels, 4 GiB buffers): pure write, copy, pure read.
Measured on the pool's B200: fill 7.50 TB/s, copy 6.65 TB/s, sum 6.51 TB/s."""
import torch
x = torch.empty(1<<30, dtype=torch.float32, device="cuda")  # 4 GiB
y = torch.empty(1<<30, dtype=torch.float32, device="cuda")
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)/n
ms=t(lambda: x.fill_(1.0)); print("fill (write only)  ", round(4.295/ms*1e3,1), "GB/s")
ms=t(lambda: y.copy_(x)); print("copy (read+write)  ", round(2*4.295/ms*1e3,1), "GB/s")
ms=t(lambda: x.sum()); print("sum  (read only)   ", round(4.295/ms*1e3,1), "GB/s")
