"""Per-launch breakdown of one config-2 step (KernelTimer, CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import tensor_core as tc
mode = sys.argv[1] if len(sys.argv) > 1 else "auto"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
qf.set_gemm_mode(mode)
if os.environ.get("QF_TC3_VARIANT"):
    from paper_1811_09599_b200 import _lib
    _lib.load().qf_tc3_set_variant(int(os.environ["QF_TC3_VARIANT"]))
if os.environ.get("QF_SMALL_ENGINE"):
    from paper_1811_09599_b200 import _lib
    _lib.load().qf_small_engine(int(os.environ["QF_SMALL_ENGINE"]))
lat = qf.Lattice.named("grid:5x5"); circ = qf.generate_rqc(lat, "1+24+1", 0)
eng = qf.AmplitudeEngine(circ, qf.grid_plan(lat, n_cuts=1))
rng = np.random.Generator(np.random.PCG64(0))
outs = [format(int(v), "025b") for v in rng.integers(0, 2 ** 25, size=nb)]
late = os.environ.get("QF_LATE", "1") != "0"
for _ in range(2): eng.amplitudes(0, outs, late=late)
with tc.KernelTimer() as kt:
    eng.amplitudes(0, outs, late=late)
torch.cuda.synchronize()
s = {}
for kind, a, b, flops, nbytes, *rest in kt.records:
    key = f"{kind} {rest[0]}  [{rest[1] if len(rest) > 1 else ''}]"
    d = s.setdefault(key, {"launches": 0, "ms": 0.0, "flops": 0, "bytes": 0})
    d["launches"] += 1; d["ms"] += a.elapsed_time(b); d["flops"] += flops; d["bytes"] += nbytes
if os.environ.get("QF_ORDER"):
    for kind, a, b, flops, nbytes, *rest in kt.records:
        print(f"ORDER {a.elapsed_time(b):7.3f} ms {kind} {rest[0]} [{rest[1] if len(rest) > 1 else ''}]")
tot = sum(d["ms"] for d in s.values())
print(f"mode={mode} batch={nb} total kernel ms {tot:.2f}")
for k, d in sorted(s.items(), key=lambda x: -x[1]["ms"])[:40]:
    print(f"{d['ms']:8.3f} ms {d['launches']:3d}x  {d['bytes']/d['ms']/1e6:7.0f} GB/s {d['flops']/d['ms']/1e9:6.1f} TF/s  {k}")
