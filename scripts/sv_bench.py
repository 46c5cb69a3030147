"""GPU state-vector simulator throughput: seeded grid RQCs 1+24+1 (complex128),
per-pass HBM traffic 2 x 16 B x 2^n against the measured HBM peak."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import statevector as sv
res = {}
for (r, c) in [(5, 5), (5, 6), (4, 8)]:
    lat = qf.Lattice.rectangle(r, c)
    circ = qf.generate_rqc(lat, "1+24+1", seed=0)
    n = circ.n
    passes = sum(len(sv.plan_passes(g, n)) for g in circ.by_cycle())
    sv.evolve_device(circ, 0); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); psi = sv.evolve_device(circ, 0); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    gbs = passes * 2 * 16 * 2 ** n / (ms / 1e3) / 1e9
    norm = float(torch.linalg.vector_norm(psi).item())
    res[f"grid:{r}x{c}"] = {"qubits": n, "passes": passes, "ms": round(ms, 2), "pass_gbs": round(gbs, 1),
                            "norm": norm, "gates": len(circ.gates)}
    print(f"grid {r}x{c} n={n}: {passes} passes, {ms:.1f} ms, {gbs:.0f} GB/s per pass, |psi|={norm:.12f}", flush=True)
    del psi; torch.cuda.empty_cache()
print(json.dumps(res))
