"""Long-K complex GEMM probe: algorithmic TFLOP/s (8*M*N*K per launch) of the
3xTF32 tensor-core engine at one shape, burst (first 5 launches) and
sustained (back to back for --seconds), with nvidia-smi clocks and power
sampled during the sustained leg; optional accuracy check vs float64.

  python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 5 [--variant V]
"""
import argparse
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1811_09599_b200 import _lib, tensor_core as tc


def sampler(idx=0):
    return subprocess.Popen(
        ["nvidia-smi", "-i", str(idx), "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
         "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE,
        stderr=subprocess.DEVNULL, text=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="8192,8192,8192")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--seconds", type=float, default=4.0)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--mode", type=int, default=2)
    ap.add_argument("--check", type=int, default=1)
    ap.add_argument("--cublas", type=int, default=0, help="also time cuBLAS TF32 fp32 matmul")
    a = ap.parse_args()
    M, N, K = (int(x) for x in a.shape.split(","))
    b = a.batch
    lib = _lib.load()
    lib.qf_tc3_set_variant(a.variant)
    g = torch.Generator(device="cuda").manual_seed(0)
    A = torch.randn(b * M * K, dtype=torch.complex64, device="cuda", generator=g)
    B = torch.randn(b * K * N, dtype=torch.complex64, device="cuda", generator=g)
    C = torch.empty(b * M * N, dtype=torch.complex64, device="cuda")
    fn = lambda: tc.gemm_buffer(b, M, N, K, A, 0, B, 0, C, mode=a.mode)
    flops = 8.0 * b * M * N * K
    fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(3):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    burst = flops * 3 / ev[0].elapsed_time(ev[1]) / 1e9
    one_ms = ev[0].elapsed_time(ev[1]) / 3
    reps = max(3, int(a.seconds * 1e3 / one_ms))
    p = sampler()
    p.stdout.readline()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    p.terminate()
    out, _ = p.communicate()
    sm, pw, rs = [], [], set()
    for line in out.splitlines():
        parts = [x.strip() for x in line.split(",")]
        try:
            sm.append(float(parts[0]))
            pw.append(float(parts[1]))
            rs.add(parts[2])
        except (ValueError, IndexError):
            pass
    sustained = flops * reps / ev[0].elapsed_time(ev[1]) / 1e9
    rec = {"shape": [b, M, N, K], "variant": a.variant, "kernel": _lib.last_kernel() if hasattr(_lib, "last_kernel") else None,
           "burst_tflops": round(burst, 1), "sustained_tflops": round(sustained, 1), "reps": reps,
           "ms_per_launch": round(ev[0].elapsed_time(ev[1]) / reps, 3),
           "sm_mhz_median": float(np.median(sm)) if sm else None,
           "power_w_median": float(np.median(pw)) if pw else None, "reasons": sorted(rs)}
    if a.check:
        rows = min(M, 64)
        Ah = A.view(b, M, K)[0, :rows].cpu().numpy().astype(np.complex128)
        Bh = B.view(b, K, N)[0].cpu().numpy().astype(np.complex128)
        want = Ah @ Bh
        got = C.view(b, M, N)[0, :rows].cpu().numpy()
        rec["rel_l2_vs_f64"] = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    if a.cublas:
        torch.backends.cuda.matmul.allow_tf32 = True
        x = torch.randn(8192, 8192, device="cuda")
        y = torch.randn(8192, 8192, device="cuda")
        for _ in range(3):
            x @ y
        torch.cuda.synchronize()
        ev[0].record()
        for _ in range(10):
            x @ y
        ev[1].record()
        torch.cuda.synchronize()
        rec["cublas_tf32_8192_tflops"] = round(2 * 8192 ** 3 * 10 / ev[0].elapsed_time(ev[1]) / 1e9, 1)
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
