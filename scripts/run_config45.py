"""Full-depth configs 4 and 5 on one B200: time a bounded set of paths
through the public engine's executor and extrapolate (labelled as such).

config 4: grid:7x7 1+40+1 seed 0, slice-first plan (2 cuts, 1024 paths),
          one bit-string, f = 1/64 (16 seeded paths)
config 5: bristlecone-70 1+32+1 seed 0, slice-first plan (4 cuts, 65536
          paths), open batch of 6 qubits (64 amplitudes), f = 0.005 (328)"""
import json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1811_09599_b200 as qf
from paper_1811_09599_b200 import tensor_core as tc
from paper_1811_09599_b200.amplitude_engine import _bits_str

which = sys.argv[1]
if os.environ.get("QF_TC3_VARIANT"):  # A/B the tensor-core kernel flavours
    from paper_1811_09599_b200 import _lib
    _lib.load().qf_tc3_set_variant(int(os.environ["QF_TC3_VARIANT"]))
max_paths = int(sys.argv[2]) if len(sys.argv) > 2 else 4
ev = lambda: torch.cuda.Event(enable_timing=True)

def timed(fn):
    a, b = ev(), ev(); a.record(); r = fn(); b.record(); torch.cuda.synchronize()
    return r, a.elapsed_time(b) / 1e3

if which == "config4":
    lat = qf.Lattice.named("grid:7x7"); circ = qf.generate_rqc(lat, "1+40+1", 0)
    plan = qf.load_plan("grid:7x7:slice-first")
    eng = qf.AmplitudeEngine(circ, plan)
    rng = np.random.Generator(np.random.PCG64(0))
    out = format(int(rng.integers(0, 2 ** 49)), "049b")
    net, t_net = timed(lambda: eng.base_net(0))
    netf = net.fix_outputs({q: int(b) for q, b in enumerate(out)})
    ex = eng._executor(netf)
    paths = qf.FidelitySpec(1 / 64, 0).paths_for(ex.cut_dims)
    open_c = ()
else:
    lat = qf.Lattice.named("bristlecone-70"); circ = qf.generate_rqc(lat, "1+32+1", 0)
    plan = qf.load_plan("bristlecone-70:slice-first")
    eng = qf.AmplitudeEngine(circ, plan)
    c_sites = tuple(sorted(plan.batch_sites[:6]))
    rng = np.random.Generator(np.random.PCG64(0))
    s_ab = "".join(str(int(b)) for b in rng.integers(0, 2, size=70))
    net, t_net = timed(lambda: eng.base_net(0))
    netf = net.fix_outputs({q: int(s_ab[q]) for q in range(70) if q not in c_sites})
    ex = eng._executor(netf)
    paths = qf.FidelitySpec(0.005, 0).paths_for(ex.cut_dims)
    open_c = c_sites
est = qf.estimate_cost(plan, lat, circ.depth, open_sites=open_c)
order = tuple(qf.network_builder.out_label(q) for q in open_c)
acc = None
times, flops = [], []
for i, p in enumerate(paths[:max_paths]):
    f0 = ex.flops
    t, dt = timed(lambda: ex.run(p))
    r = t.transpose_to(order) if order else t
    acc = r.data.clone() if acc is None else acc + r.data
    times.append(dt); flops.append(ex.flops - f0)
    print(f"path {i} {p}: {dt:.2f} s, {(ex.flops - f0) / 1e12:.2f} TFLOP, "
          f"{(ex.flops - f0) / dt / 1e12:.1f} TFLOP/s", flush=True)
    if i == 0:
        with tc.KernelTimer() as kt:
            ex._steps.clear(); ex._sites.clear(); ex.run(p)
        for k, d in sorted(kt.summary(detail=True).items(), key=lambda x: -x[1]["ms"])[:14]:
            print(f"   {k}: {d['ms']:.1f} ms, {d['launches']} launches, "
                  f"{d['flops'] / d['ms'] / 1e9 if d['ms'] else 0:.1f} TFLOP/s, {d['bytes'] / d['ms'] / 1e6:.0f} GB/s")
vals = acc.cpu().numpy()
n_units = 1 if which == "config4" else 64
steady = times[1:] or times
proj = times[0] + np.mean(steady) * (len(paths) - 1)
res = {"config": which, "paths_total": est.paths, "paths_selected": len(paths),
       "paths_timed": len(times), "network_build_s": round(t_net, 2),
       "first_path_s": round(times[0], 2), "steady_path_s": round(float(np.mean(steady)), 3),
       "executed_tflops_per_s": round(sum(flops) / sum(times) / 1e12, 1),
       "projected_unit_s": round(float(proj), 1),
       "projected_amplitudes_per_s_1gpu": round(n_units / proj, 4),
       "algorithmic_flops_per_unit": est.total_flops * len(paths) // est.paths,
       "partial_sum_finite": bool(np.isfinite(vals).all()),
       "partial_norm2_x_2^n": float(np.sum(np.abs(vals) ** 2) * 2 ** circ.n / max(1, vals.size)),
       "note": "projection = first path + mean(later paths) x remaining selected paths"}
print(json.dumps(res))
