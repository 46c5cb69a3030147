"""Config-4 paths with / without TMA views of compute-bound operands."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import tensor_core as tc
which = sys.argv[1] if len(sys.argv) > 1 else "config4"
rng = np.random.Generator(np.random.PCG64(0))
if which == "config4":
    lat = qf.Lattice.named("grid:7x7"); circ = qf.generate_rqc(lat, "1+40+1", 0)
    eng = qf.AmplitudeEngine(circ, qf.load_plan("grid:7x7:slice-first"))
    out = format(int(rng.integers(0, 2 ** 49)), "049b")
    net = eng.base_net(0).fix_outputs({q: int(b) for q, b in enumerate(out)})
    f = 1 / 64
else:
    lat = qf.Lattice.named("bristlecone-70"); circ = qf.generate_rqc(lat, "1+32+1", 0)
    plan = qf.load_plan("bristlecone-70:slice-first")
    eng = qf.AmplitudeEngine(circ, plan)
    c_sites = tuple(sorted(plan.batch_sites[:6]))
    s_ab = "".join(str(int(b)) for b in rng.integers(0, 2, size=70))
    net = eng.base_net(0).fix_outputs({q: int(s_ab[q]) for q in range(70) if q not in c_sites})
    f = 0.005
for mode in (os.environ.get("MODES", "compute-views,no-compute-views,compute-views,no-compute-views").split(",")):
    tc._compute_views = mode == "compute-views"
    ex = eng._executor(net)
    paths = qf.FidelitySpec(f, 0).paths_for(ex.cut_dims)
    ex.run(paths[0]); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 6
    for p in paths[1:1 + n]:
        ex.run(p)
    b.record(); torch.cuda.synchronize()
    print(which, mode, round(a.elapsed_time(b) / n, 2), "ms per path", flush=True)
    del ex
    torch.cuda.empty_cache()
