"""Benchmark: RQC amplitudes/s on the B200 (BASELINE.json metric).

Headline workload (default `--workload config4`, the largest single-GPU
config of BASELINE.json and the tensor-core-bound one): seeded grid:7x7
random circuit, depth 1+40+1 (bond dim 32), the reference's two cuts
(1024 slices) in a slice-first plan, fidelity f = 1/64 (16 seeded paths per
amplitude), 256 seeded bit-strings.  One *step* = one contraction path on
every rank (`PlanExecutor.run`); value = amplitudes/s = paths/s / 16.  Short
runs of the other configs (2, 1, 3 and 5) are reported under `secondary`.

Config 2 (`--workload config2`, BASELINE configs[1]): seeded grid:5x5
random circuit, depth 1+24+1 (bond dim 8), 1024 seed-drawn output
bit-strings, plan grid_plan(lattice, n_cuts=1) -- one cut of dimension 8
across the middle column (8 slices).  One *step* = all 1024 amplitudes
(every slice of every bit-string).

  value  : amplitudes/s with inputs resident in HBM (device-timed, CUDA
           events on the launching stream, max over ranks).
  e2e    : the same through the public API `AmplitudeEngine.amplitudes`
           with host bit-strings in and host amplitudes out every step.
  roofline / kernels : the dominant kernel's achieved rate from per-launch
           CUDA events (tensor_core.KernelTimer) in a separate profiled step.
  cpu_baseline : the CPU oracle port (oracle/rqc_oracle.py, the reference
           algorithm restated in numpy) on a bounded sample, all host cores.

Multi-GPU (torchrun, one process per GPU): `--shard bitstrings` (default,
weak scaling: each rank computes its own 1024 bit-strings, no collective);
`--shard slices` (the config as stated: the 8 slices are split across
ranks and the partial amplitudes all-reduced over NCCL, strong scaling).

`--impl reference` times the reference's algorithm on the host cores (the
oracle port, multi-process) for the same metric/config.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

SEED = 0
# (lattice, depth, grid_plan n_cuts, bit-strings per step, description, L2 note)
WORKLOADS = {
    "config2": ("grid:5x5", "1+24+1", 1, 1024,
                "config2: grid:5x5 RQC 1+24+1 (bond 8), 1024 bitstrings/rank, grid_plan n_cuts=1 "
                "(8 slices of dim-8 cut)",
                "working set > L2 (126 MB): 1024 x 2^18-entry intermediates per step"),
    "config1": ("grid:4x4", "1+16+1", 0, 64,
                "config1: grid:4x4 RQC 1+16+1 (bond 4), 64 bitstrings/rank, no cuts",
                "working set < L2 (launch-bound workload; inputs re-gathered every step)"),
}
N_BITSTRINGS = WORKLOADS["config2"][3]
LATTICE, DEPTH, N_CUTS = WORKLOADS["config2"][:3]


def workload_config(shard: str, world: int, workload: str = "config2") -> dict:
    lat, depth, cuts, nb, desc, l2 = WORKLOADS[workload]
    return {"workload": desc, "lattice": lat, "depth": depth, "circuit_seed": SEED, "cuts": cuts,
            "bitstrings_per_step": nb * (world if shard == "bitstrings" else 1),
            "parallelism": f"{shard}-sharded x{world}", "l2": l2}


def bitstrings(rank: int, n: int, count: int) -> list:
    rng = np.random.Generator(np.random.PCG64(SEED + rank))
    return [format(int(v), f"0{n}b") for v in rng.integers(0, 2 ** n, size=count)]


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port on host cores (never the product)


def _oracle_worker(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    circuit_text, plan_text, outs = args
    from oracle import rqc_oracle
    eng = rqc_oracle.OracleEngine(circuit_text, plan_text, np.complex64)
    t0 = time.perf_counter()
    for o in outs:
        eng.amplitude(0, o)
    return time.perf_counter() - t0


def cpu_oracle_rate(circuit_text: str, plan_text: str, outs: list, procs: int,
                    of: str = "the 1024 config-2 bit-strings") -> dict:
    """Amplitudes/s of the numpy oracle with `procs` single-threaded worker
    processes (spawned with every BLAS/OpenMP pool pinned to 1 thread)."""
    import multiprocessing as mp
    env_keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in env_keys}
    for k in env_keys:
        os.environ[k] = "1"
    try:
        ctx = mp.get_context("spawn")
        chunks = [outs[i::procs] for i in range(procs)]
        chunks = [c for c in chunks if c]
        with ctx.Pool(len(chunks)) as pool:
            pool.map(_oracle_worker, [(circuit_text, plan_text, c[:1]) for c in chunks])  # warm
            t0 = time.perf_counter()
            pool.map(_oracle_worker, [(circuit_text, plan_text, c) for c in chunks])
            wall = time.perf_counter() - t0
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return {"value": len(outs) / wall, "unit": "amplitudes/s", "cores": len(chunks),
            "kind": "port", "seconds": wall,
            "sample": f"{len(outs)} of {of}, oracle/rqc_oracle.py "
                      f"(numpy restatement of the reference), {len(chunks)} processes x 1 thread"}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# distributed plumbing


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def init_dist(world: int, backend: str):
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend)
    return dist


def max_over_ranks(x: float, world: int, device=None) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            # nvidia-smi takes ~0.1-0.5 s to start: block until it samples, so a
            # timed region of a few tens of ms is still covered (20 ms period)
            self.first = self.proc.stdout.readline()
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in [getattr(self, "first", "")] + out.splitlines() if l.strip()]
        return False

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in getattr(self, "lines", []):
            parts = [p.strip() for p in line.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except (ValueError, IndexError):
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# the GPU arm


def measured_traffic(workload: str, kernel: str, algorithmic_per_step: float, launches: int):
    """DRAM bytes (read + write) of `kernel` over one step from the committed
    ncu capture (profiles/traffic_<workload>.json, made by
    scripts/make_traffic_json.py), beside the algorithmic bytes of the same
    step; per launch = per step / the launches this bench times (a kernel
    timed as one record may be several ncu launches).  None when no capture
    of this workload/kernel is committed."""
    path = os.path.join(ROOT, "profiles", f"traffic_{workload}.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        rec = json.load(fh).get("kernels", {}).get(kernel)
    if rec is None:
        return None
    dram = rec["dram_read"] + rec["dram_write"]
    if launches <= 0:   # path workloads: the capture's own launch count (one path)
        launches = rec["launches"]
        algorithmic_per_step *= launches
    return {"dram_bytes_per_step": round(dram), "algorithmic_bytes_per_step": round(algorithmic_per_step),
            "dram_bytes_per_launch": round(dram / max(launches, 1)),
            "ratio": round(dram / max(algorithmic_per_step, 1), 3),
            "source": f"profiles/traffic_{workload}.json (ncu dram__bytes_read.sum + "
                      f"dram__bytes_write.sum over {rec['launches']} ncu launches of one step)"}


def tensor_pipe_ncu(kernel: str):
    """sm__pipe_tensor_cycles_active of `kernel` from the committed ncu
    --set full capture (profiles/tensor_pipe.json: a separate, unthrottled
    single-launch run -- context for the live `tensor_pipe_util`, not a
    measurement of this run)."""
    path = os.path.join(ROOT, "profiles", "tensor_pipe.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh).get(kernel)


def peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        d["source"] = "MEASURED_PEAKS.json (measured)"
    else:
        d = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
             "source": "B200_PROFILING.md fallback"}
    return d


def run_gpu(args):
    import torch

    import paper_1811_09599_b200 as qf
    from paper_1811_09599_b200 import _lib
    from paper_1811_09599_b200 import tensor_core as tc

    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    if args.gemm:
        qf.set_gemm_mode(args.gemm)

    LATTICE, DEPTH, N_CUTS, N_BITSTRINGS = WORKLOADS[args.workload][:4]
    lat = qf.Lattice.named(LATTICE)
    circ = qf.generate_rqc(lat, DEPTH, SEED)
    plan = qf.grid_plan(lat, n_cuts=N_CUTS)
    shard = args.shard
    group = None
    if shard == "slices" and world > 1:
        import torch.distributed as dist
        group = dist.group.WORLD
    eng = qf.AmplitudeEngine(circ, plan, device=local, group=group)
    outs = bitstrings(rank if shard == "bitstrings" else 0, circ.n, N_BITSTRINGS)
    bits_host = torch.tensor([[int(c) for c in o] for o in outs], dtype=torch.int32).pin_memory()
    # ---- device-resident step (value) ----
    base = eng.base_net(0)
    dev_bits = bits_host
    if args.late:   # the order amplitudes() walks a late-sliced batch in (host sort)
        dev_bits = bits_host[torch.from_numpy(eng.batch_order(bits_host.numpy()))]
    bits_dev = dev_bits.t().contiguous().to(dev)        # (sites, B): row j = bits of site j

    runner = (eng._graph_runner(0, N_BITSTRINGS, qf.FidelitySpec(), args.late) if args.graph
              else None)
    from paper_1811_09599_b200.amplitude_engine import _finisher

    def batched_net():
        if args.late:
            return base.late_outputs(bits_dev, tuple(range(circ.n)))
        return base.fix_outputs_batch_device(bits_dev, tuple(range(circ.n)))

    def step_device():
        if runner is not None:           # captured plan walk, bits already resident
            acc = runner.replay_device(bits_dev)
            qf.reduce_partials(acc, group)
            return acc
        net = batched_net()
        ex = eng._executor(net)
        paths = qf.FidelitySpec().paths_for(ex.cut_dims)
        acc, _ = eng._sum_paths(ex, paths, _finisher(net), N_BITSTRINGS)
        return acc

    def step_e2e():
        res, _ = eng.amplitudes(0, outs, graph=args.graph, late=args.late)
        return res

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    _lib.launch_count(reset=True)
    barrier(world)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        start.record()
        for _ in range(args.steps):
            acc = step_device()
        end.record()
        torch.cuda.synchronize()
    barrier(world)
    launches = _lib.launch_count(reset=True) // max(args.steps, 1)
    if runner is not None:
        launches = runner.kernels          # kernels recorded in the replayed graph
    ms = max_over_ranks(start.elapsed_time(end) / args.steps, world, dev)
    amps_per_step = N_BITSTRINGS * (world if shard == "bitstrings" else 1)
    value = amps_per_step / (ms / 1e3)

    # ---- N>1 self-check: the sharded result equals an unsharded (group=None)
    # recomputation of this rank's bit-strings
    selfcheck = None
    if world > 1:
        got = acc[:N_BITSTRINGS].cpu().numpy()
        if args.late:
            back = np.empty_like(got)
            back[eng.batch_order(bits_host.numpy())] = got
            got = back
        solo = qf.AmplitudeEngine(circ, plan, device=local)
        want, _ = solo.amplitudes(0, outs)
        err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
        selfcheck = {"what": f"rank's {N_BITSTRINGS} amplitudes ({shard}-sharded x{world}) vs an "
                             f"unsharded recomputation", "rel_l2": err, "ok": err < 1e-4}
        if err >= 1e-4:
            raise AssertionError(f"N>1 self-check failed on rank {rank}: {selfcheck}")

    # ---- end-to-end through the public API (host in, host out) ----
    for _ in range(max(1, args.warmup // 2)):
        step_e2e()
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(args.steps):
        res = step_e2e()
    e1.record()
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1) / args.steps, wall_ms), world, dev)
    e2e = amps_per_step / (e2e_ms / 1e3)

    # ---- the reference's single-call API as a drop-in user calls it: one
    # amplitude() per bit-string (rq/amplitude_engine.py:114-126), host wall
    # time; after the first (eager) call the engine replays a captured walk
    single = None
    if rank == 0 and world == 1:
        n_single = min(64, len(outs))
        for o in outs[:4]:
            eng.amplitude(0, o)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for o in outs[:n_single]:
            eng.amplitude(0, o)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / n_single
        single = {"value": round(1.0 / dt, 1), "unit": "amplitudes/s", "ms_per_call": round(dt * 1e3, 3),
                  "calls": n_single,
                  "api": "AmplitudeEngine.amplitude(0, bits) per bit-string, host wall time"}

    # ---- per-kernel profile (one extra, separately timed, eager step) ----
    with tc.KernelTimer() as kt:
        net = batched_net()
        ex = eng._executor(net)
        eng._sum_paths(ex, qf.FidelitySpec().paths_for(ex.cut_dims), _finisher(net),
                       N_BITSTRINGS)
    kinds = kt.summary()
    kerns = kt.summary(by_kernel=True)
    exec_flops = sum(d["flops"] for d in kinds.values())   # GEMM flops actually issued
    stats_flops = qf.estimate_cost(plan, lat, DEPTH).total_flops  # per amplitude
    pk = peaks()
    result = None
    if rank == 0:
        ops, kern = {}, {}
        total = sum(d["ms"] for d in kinds.values()) or 1.0
        for kind, d in kinds.items():
            ops[kind] = {"launches": d["launches"], "ms": round(d["ms"], 4),
                         "share": round(d["ms"] / total, 4)}
        for name, d in kerns.items():
            kern[name] = {"launches": d["launches"], "ms": round(d["ms"], 4),
                          "share": round(d["ms"] / total, 4),
                          "tflops": round(d["flops"] / d["ms"] / 1e9, 2) if d["ms"] else None,
                          "gbs": round(d["bytes"] / d["ms"] / 1e6, 1) if d["ms"] else None}
        # 3xTF32 complex ceiling of the real-block kernel (TF32 = burst bf16 / 2:
        # a config-2 step is milliseconds long); the ridge classifies launches
        tensor_peak, _, peak_basis = tensor_peak_of(pk, sustained=False)
        ridge = tensor_peak * 1e12 / (pk["hbm_gbs"] * 1e9)
        # launches grouped by (CUDA kernel, the roofline that bounds the
        # launch's shape: tensor if its algorithmic flop/byte >= the ridge);
        # the dominant group is the one with the most time in the step
        groups = {}
        for kind, a, b, flops, nbytes, *rest in kt.records:
            name = rest[1] if len(rest) > 1 and rest[1] else kind
            bnd = "tensor" if flops and "tc3" in name and flops / max(nbytes, 1) >= ridge else "hbm"
            g = groups.setdefault((name, bnd), {"launches": 0, "ms": 0.0, "flops": 0, "bytes": 0})
            g["launches"] += 1
            g["ms"] += a.elapsed_time(b)
            g["flops"] += flops
            g["bytes"] += nbytes

        def roof_of(key):
            name, bnd = key
            g = groups[key]
            if bnd == "tensor":
                peak, _, basis = tensor_peak_of(pk, sustained=False, kernel=name)
                achieved = g["flops"] / g["ms"] / 1e9
                r = {"bound": "tensor", "unit": "TFLOP/s", "kernel": name, "peak_basis": basis}
            else:
                achieved, peak = g["bytes"] / g["ms"] / 1e6, pk["hbm_gbs"]
                r = {"bound": "hbm", "unit": "GB/s", "kernel": name,
                     "peak_basis": f"hbm_gbs {pk['source']}"}
            r.update({"achieved": round(achieved, 2), "peak": round(peak, 1),
                      "frac": round(achieved / peak, 4), "launches": g["launches"],
                      "ms": round(g["ms"], 4),
                      "arithmetic_intensity": round(g["flops"] / max(g["bytes"], 1), 2)})
            return r

        dkey = max(groups, key=lambda k: groups[k]["ms"])
        dom, d = dkey[0], groups[dkey]
        roof = roof_of(dkey)
        fam = kerns.get(dom, d)
        roof.update({"traffic_detail": measured_traffic(args.workload, dom, fam["bytes"],
                                                        fam["launches"]),
                     "ridge": round(ridge, 2),
                     "algorithmic": (f"{dom} launches whose shape is {dkey[1]}-bound (flop/byte "
                                     f"{'>=' if dkey[1] == 'tensor' else '<'} ridge): 8*m*k*n "
                                     f"flops and 8*(m*k + k*n + m*n)*batch bytes per launch, "
                                     f"summed over the {d['launches']} such launches of one step, "
                                     f"/ their CUDA-event time"),
                     "other_bound": [roof_of(k) for k in sorted(groups, key=lambda k: -groups[k]["ms"])
                                     if k != dkey and k[0] == dom]})
        # DRAM bytes per launch over the whole kernel family (ncu cannot split it by bound)
        roof["traffic"] = (roof["traffic_detail"] or {}).get("dram_bytes_per_launch")
        clk = clocks.summary()
        cpu = None
        if not args.no_cpu_baseline:
            sample = max(8, min(len(outs), int(args.cpu_sample)))
            cpu = cpu_oracle_rate(qf.write_circuit(circ), qf.format_plan(plan), outs[:sample],
                                  host_cores(), f"the {len(outs)} {args.workload} bit-strings")
        result = {
            "metric": "amplitudes/s", "value": round(value, 2), "unit": "amplitudes/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak" if shard == "bitstrings" else "strong",
            "vs_baseline": None, "dtype": "c64 (fp32 complex; 3xTF32 on tensor cores)",
            "data": "synthetic (seeded RQC + seeded bit-strings; the paper's circuit files are "
                    "not in the container)",
            "config": workload_config(shard, world, args.workload),
            "cuda_graph": bool(args.graph),
            "sustained_tflops": round(amps_per_step * stats_flops / (ms / 1e3) / 1e12, 3),
            "flops_per_amplitude": stats_flops,
            "late_output_slicing": bool(args.late),
            "executed_flops_per_step": int(exec_flops),
            "executed_tflops": round(exec_flops * (amps_per_step // N_BITSTRINGS) / (ms / 1e3)
                                     / 1e12, 3),
            "gemm_mode": qf.get_gemm_mode(),
            "e2e": {"value": round(e2e, 2), "unit": "amplitudes/s",
                    "h2d_bytes_per_step": int(bits_host.numel() * 4),
                    "d2h_bytes_per_step": int(amps_per_step // world * 8),
                    "api": "AmplitudeEngine.amplitudes(0, host bit-strings) -> host ndarray"},
            "roofline": roof, "kernels": kern, "ops": ops, "gpu_launches": int(launches),
            "clocks": clk, "cpu_baseline": cpu, "self_check": selfcheck,
            "single_call": single,
        }
    barrier(world)
    return result


def config3_cases(log2n: int, count: int, seed: int):
    """Config 3: `count` seeded permutations of a 2^log2n complex64 tensor;
    first half all-binary dims, second half mixed 2/4/8/16 dims (rank >= 10)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cases = []
    for i in range(count):
        if i < count // 2:
            dims = [2] * log2n
        else:
            while True:
                bits, tot = [], 0
                while tot < log2n:
                    b = min(int(rng.integers(1, 5)), log2n - tot)
                    bits.append(b)
                    tot += b
                if len(bits) >= 10:
                    break
            dims = [1 << b for b in bits]
        cases.append((dims, [int(p) for p in rng.permutation(len(dims))]))
    return cases


def run_permute(args):
    """BASELINE config 3: K1 permutation GB/s at 2^24 / 2^28 / 2^30 elements
    (16 bytes per element: 8 read + 8 written)."""
    import torch

    from paper_1811_09599_b200 import _lib
    from paper_1811_09599_b200 import tensor_core as tc

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    pk = peaks()
    sizes = [int(s) for s in args.perm_sizes.split(",")]
    per_size = {}
    eager = {s: [] for s in sizes}
    launches = 0
    for log2n in sizes:
        n = 1 << log2n
        src = torch.randn(n, dtype=torch.complex64, device="cuda")
        dst = torch.empty_like(src)
        rates = {"binary": [], "mixed": []}
        for i, (dims, perm) in enumerate(config3_cases(log2n, args.perms, seed=log2n)):
            for _ in range(args.warmup):
                tc.permute_buffer(src, dims, perm, out=dst)
            torch.cuda.synchronize()
            _lib.launch_count(reset=True)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.steps):
                tc.permute_buffer(src, dims, perm, out=dst)
            b.record()
            torch.cuda.synchronize()
            launches += _lib.launch_count(reset=True)
            ms = a.elapsed_time(b) / args.steps
            eager[log2n].append(16 * n / ms / 1e6)
            if args.perm_graph:
                # the K launches replayed from one CUDA graph: no host gaps
                # between back-to-back 40-60 us launches at 2^24
                g = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream()
                cs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
                    for _ in range(args.steps):
                        tc.permute_buffer(src, dims, perm, out=dst)
                torch.cuda.current_stream().wait_stream(cs)
                _lib.launch_count(reset=True)
                g.replay()
                torch.cuda.synchronize()
                a.record()
                g.replay()
                b.record()
                torch.cuda.synchronize()
                launches += args.steps
                ms = a.elapsed_time(b) / args.steps
                del g
            rates["binary" if i < args.perms // 2 else "mixed"].append(16 * n / ms / 1e6)
            if i in (0, args.perms // 2):  # spot-check bytes against index arithmetic
                idx = torch.randint(0, n, (4096,), device="cuda")
                out_dims = [dims[p] for p in perm]
                strides = [int(np.prod(dims[j + 1:])) for j in range(len(dims))]
                rem = idx.clone()
                src_idx = torch.zeros_like(idx)
                for j in range(len(out_dims) - 1, -1, -1):
                    src_idx += (rem % out_dims[j]) * strides[perm[j]]
                    rem //= out_dims[j]
                if not torch.equal(dst[idx], src[src_idx]):
                    raise AssertionError(f"permutation mismatch at 2^{log2n} {dims} {perm}")
        per_size[f"2^{log2n}"] = {k: {"mean_gbs": round(float(np.mean(v)), 1),
                                      "min_gbs": round(float(np.min(v)), 1),
                                      "max_gbs": round(float(np.max(v)), 1),
                                      "frac_mean": round(float(np.mean(v)) / pk["hbm_gbs"], 4)}
                                  for k, v in rates.items() if v}
        per_size[f"2^{log2n}"]["eager_mean_gbs"] = round(float(np.mean(eager[log2n])), 1)
        del src, dst
        torch.cuda.empty_cache()
    allv = [d["mean_gbs"] for s in per_size.values() for d in s.values() if isinstance(d, dict)]
    value = float(np.mean(allv))
    return {"metric": "permutation GB/s (config 3)", "value": round(value, 1), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c64",
            "data": "synthetic i.i.d. complex normal", "config": {
                "workload": f"config3: {args.perms} seeded perms per size "
                            f"(half binary dims, half mixed 2/4/8/16), sizes 2^{sizes}",
                "l2": "inputs larger than L2 (>= 256 MiB)",
                "timing": "K launches replayed from one CUDA graph" if args.perm_graph
                          else "K eager launches"},
            "roofline": {"bound": "hbm", "unit": "GB/s", "kernel": "permute_tiled",
                         "achieved": round(value, 1), "peak": pk["hbm_gbs"],
                         "frac": round(value / pk["hbm_gbs"], 4), "traffic": None,
                         "algorithmic": "16 B per element (8 read + 8 written) per launch"},
            "per_size": per_size, "gpu_launches": int(launches)}


# ---------------------------------------------------------------------------
# configs 4 and 5 at full depth: one step = one contraction path


PATH_WORKLOADS = {
    "config4": {
        "lattice": "grid:7x7", "depth": "1+40+1", "plan": "grid:7x7:slice-first", "f": 1 / 64, "open": 0,
        "units": 256, "amps_per_unit": 1, "cpu_depth": "1+28+1",
        "desc": "config4: grid:7x7 RQC 1+40+1 (bond 32), slice-first plan with the reference's "
                "cuts (right 19:26, bottom 37:38; 1024 slices), f=1/64 (16 seeded paths per "
                "amplitude), 256 seeded bit-strings walked in order",
    },
    "config4f1": {
        "lattice": "grid:7x7", "depth": "1+40+1", "plan": "grid:7x7:slice-first", "f": 1.0, "open": 0,
        "units": 256, "amps_per_unit": 1, "cpu_depth": "1+28+1",
        "desc": "config4 at f=1: grid:7x7 RQC 1+40+1 (bond 32), slice-first plan with the "
                "reference's cuts (right 19:26, bottom 37:38), all 1024 slices per amplitude in "
                "lexicographic order (reuse=outer steps cached across consecutive paths), 256 "
                "seeded bit-strings walked in order",
    },
    "config5": {
        "lattice": "bristlecone-70", "depth": "1+32+1", "plan": "bristlecone-70:slice-first", "f": 0.005,
        "open": 6, "units": 1000, "amps_per_unit": 64, "cpu_depth": "1+24+1",
        "desc": "config5: bristlecone-70 RQC 1+32+1 (bond 16), slice-first plan with the "
                "reference's cuts w0..w3 (65536 slices), f=0.005 (328 seeded paths per batch), "
                "6 open qubits (64 amplitudes per batch), 1000 seeded s_AB batches",
    },
}


def path_units(wl: dict, circ, plan, count: int) -> list:
    """The workload's seeded units: output bit-strings (config 4) or s_AB
    strings of the open-qubit batches (config 5), as {qubit: bit} fixings."""
    rng = np.random.Generator(np.random.PCG64(SEED))
    n = circ.n
    c_sites = tuple(sorted(plan.batch_sites[:wl["open"]])) if wl["open"] else ()
    units = []
    for v in rng.integers(0, 2 ** min(n, 62), size=count):
        bits = format(int(v), f"0{n}b")[-n:] if n <= 62 else None
        if bits is None:   # > 62 qubits: draw the string bit by bit
            bits = "".join(str(int(b)) for b in rng.integers(0, 2, size=n))
        units.append((bits, {q: int(bits[q]) for q in range(n) if q not in c_sites}))
    return units, c_sites


def tensor_peak_of(pk: dict, sustained: bool, kernel: str = "cgemm_tc3k") -> tuple:
    """(3xTF32 complex ceiling in algorithmic TFLOP/s, TF32 peak, basis) from
    the driver-measured bf16 peak: TF32 dense runs at half the bf16 rate, and
    the kernel issues `mma_per_cmac` real TF32 MMAs of k-width 1 per complex
    MAC (8 algorithmic flops)."""
    from paper_1811_09599_b200 import tensor_core as tc
    bf16 = pk["bf16_tflops_sustained"] if sustained else pk["bf16_tflops"]
    tf32 = bf16 / 2
    per = tc.tc3_real_macs_per_complex_mac(kernel)
    return (tf32 * 8 / (2 * per), tf32,
            f"{'bf16_tflops_sustained' if sustained else 'bf16_tflops'} {bf16} ({pk['source']}) "
            f"/ 2 = TF32 {tf32:.1f}; x 8 / (2 x {per} real TF32 MACs per complex MAC)")


def sm_count_of(torch) -> int:
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def gemm_engines_4096(torch, tc, _lib) -> dict:
    """Algorithmic TFLOP/s (8*M*N*K) of the FFMA kernel and of the 3xTF32
    tensor-core kernel on the same 4096^3 complex64 GEMM, 3 launches each
    after a warm-up, CUDA events."""
    n = 4096
    g = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn(n * n, dtype=torch.complex64, device="cuda", generator=g)
    B = torch.randn(n * n, dtype=torch.complex64, device="cuda", generator=g)
    C = torch.empty(n * n, dtype=torch.complex64, device="cuda")
    out = {}
    for name, mode in (("ffma_tflops", _lib.GEMM_FFMA), ("tc3_tflops", _lib.GEMM_TC3)):
        tc.gemm_buffer(1, n, n, n, A, 0, B, 0, C, mode=mode)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            tc.gemm_buffer(1, n, n, n, A, 0, B, 0, C, mode=mode)
        b.record()
        torch.cuda.synchronize()
        out[name] = round(8.0 * n ** 3 * 3 / a.elapsed_time(b) / 1e9, 1)
        out[name.replace("_tflops", "_kernel")] = _lib.last_kernel()
    # the FP32 SIMT ceiling the FFMA kernel is measured against: cuBLAS SGEMM
    # with TF32 off (a library GEMM as a yardstick, not part of the path)
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        x = torch.randn(8192, 8192, device="cuda", generator=g)
        y = torch.randn(8192, 8192, device="cuda", generator=g)
        x @ y
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            x @ y
        b.record()
        torch.cuda.synchronize()
        out["fp32_simt_sgemm_tflops"] = round(2.0 * 8192 ** 3 * 3 / a.elapsed_time(b) / 1e9, 1)
        out["ffma_frac_of_fp32_simt"] = round(out["ffma_tflops"] / out["fp32_simt_sgemm_tflops"], 3)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev
    return out


def run_paths(args):
    """Configs 4/5 at full depth.  One step = one contraction path of the
    current unit on every rank (PlanExecutor.run, the reference's public
    per-path call, rq/contraction_plan.py:477); a unit's selected paths are
    split contiguously over the ranks and its partial sum is all-reduced
    (slices.reduce_partials) when the unit completes.  `value` = amplitudes/s
    with the network resident in HBM; `e2e` = AmplitudeEngine.amplitude /
    amplitude_batch (host circuit + bits in, host amplitudes out, network
    built per call)."""
    import torch

    import paper_1811_09599_b200 as qf
    from paper_1811_09599_b200 import _lib
    from paper_1811_09599_b200 import tensor_core as tc
    from paper_1811_09599_b200 import plan_tools as pt
    from paper_1811_09599_b200.network_builder import out_label

    rank, world, local = dist_env()
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        import torch.distributed as dist
        group = dist.group.WORLD
    if args.gemm:
        qf.set_gemm_mode(args.gemm)
    wl = PATH_WORKLOADS[args.workload]
    lat = qf.Lattice.named(wl["lattice"])
    circ = qf.generate_rqc(lat, wl["depth"], SEED)
    plan = qf.load_plan(wl["plan"])
    fid = qf.FidelitySpec(wl["f"], SEED)
    units, c_sites = path_units(wl, circ, plan, wl["units"])
    order = tuple(out_label(q) for q in c_sites)
    width = 2 ** len(c_sites)
    eng = qf.AmplitudeEngine(circ, plan, device=local)
    base = eng.base_net(0)
    n_paths = len(fid.paths_for(plan.cut_dims(base.bond_dim)))
    per_rank = -(-n_paths // world)            # steps per unit on every rank (max shard)
    flops_unit = pt.fidelity_flops(plan, lat, wl["depth"], wl["f"], SEED,
                                   open_sites=c_sites)
    state = {"u": 0, "i": 0, "ex": None, "mine": None, "acc": None, "results": [],
             "contrib": {}}

    def start_unit():
        bits, fixed = units[state["u"] % len(units)]
        net = base.fix_outputs(fixed)
        ex = qf.PlanExecutor(net, plan)
        paths = fid.paths_for(ex.cut_dims)
        state.update(ex=ex, mine=qf.SliceShard(rank, world).take(paths), i=0,
                     acc=torch.zeros(width, dtype=torch.complex64, device=dev))

    def step():
        if state["ex"] is None:
            start_unit()
        i = state["i"]
        if i < len(state["mine"]):
            p = state["mine"][i]
            t = state["ex"].run(p)
            t = t.transpose_to(order) if order else t
            tc.accumulate_buffer(t.data, state["acc"], width)
            if state["u"] == 0 and i == 0:
                state["contrib"] = {"path": tuple(p), "value": t.data[:width].clone()}
        state["i"] += 1
        if state["i"] == per_rank:              # unit done on every rank: one collective
            qf.reduce_partials(state["acc"], group)
            state["results"].append(state["acc"])
            state["u"] += 1
            state["ex"] = None

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    _lib.launch_count(reset=True)
    barrier(world)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks, tc.KernelTimer() as kt:
        start.record()
        for _ in range(args.steps):
            step()
        end.record()
        torch.cuda.synchronize()
    barrier(world)
    launches = _lib.launch_count(reset=True)
    ms = max_over_ranks(start.elapsed_time(end) / args.steps, world, dev)
    paths_per_s = world * 1e3 / ms * min(1.0, n_paths / (per_rank * world))
    value = paths_per_s / n_paths * wl["amps_per_unit"]

    # dominant kernel over the timed region (events on the launching stream)
    kerns = kt.summary(by_kernel=True)
    dom = max(kerns, key=lambda k: kerns[k]["ms"])
    d = kerns[dom]
    step_kernel_ms = sum(x["ms"] for x in kerns.values())
    exec_flops = sum(x["flops"] for x in kerns.values())
    pk = peaks()
    # The ceiling is the BURST bf16 figure / 2 (TF32): the long-K kernels run
    # on the 1 kW power cap, and the wide kernel sustains MORE TF32 MMA work
    # under that cap than the sustained cuBLAS bf16 figure / 2 predicts
    # (fraction 1.03-1.08 of it), so the sustained figure is not a ceiling for
    # this instruction mix; its fraction is printed beside the main one, and
    # so is the pipe utilisation at the SM clock measured under load
    # (2048 TF32 MACs/clk/SM, scripts/micro/tc_rate.cu).
    ceil, tf32, basis = tensor_peak_of(pk, sustained=False, kernel=dom)
    ceil_s, tf32_s, _ = tensor_peak_of(pk, sustained=True, kernel=dom)
    achieved = d["flops"] / d["ms"] / 1e9
    per = tc.tc3_real_macs_per_complex_mac(dom)
    roof = {"bound": "tensor", "unit": "TFLOP/s", "kernel": dom,
            "achieved": round(achieved, 2), "peak": round(ceil, 1),
            "frac": round(achieved / ceil, 4), "peak_basis": basis,
            "launches": d["launches"], "ms_per_step": round(d["ms"] / args.steps, 2),
            "share_of_step": round(d["ms"] / args.steps / ms, 4),
            "tensor_pipe_util": round(achieved * 2 * per / 8 / tf32, 4),
            "frac_of_sustained_bf16_derived_ceiling": round(achieved / ceil_s, 4),
            "frac_of_real_block_3xtf32_ceiling": round(achieved / (tf32 / 3), 4),
            "algorithmic": f"8*m*k*n flops per {dom} launch summed over the {d['launches']} launches "
                           f"of the {args.steps} timed steps / their CUDA-event time (eager launches, "
                           f"events on the launching stream)",
            "traffic_detail": measured_traffic(args.workload, dom, d["bytes"] / max(d["launches"], 1), 0)}
    roof["traffic"] = (roof["traffic_detail"] or {}).get("dram_bytes_per_launch")
    ncu_pipe = tensor_pipe_ncu(dom)
    if ncu_pipe:
        roof["tensor_pipe_active_ncu"] = ncu_pipe

    # ---- the plain FFMA engine (K3) beside the tensor-core engine on one
    # 4096^3 complex GEMM (outside the timed region; rank 0)
    if rank == 0:
        roof["ffma_vs_tensor_4096"] = gemm_engines_4096(torch, tc, _lib)

    # ---- N>1 self-check: rank 0 recomputes the first path another rank walked
    selfcheck = None
    if world > 1:
        import torch.distributed as dist
        gathered = [None] * world
        c = state["contrib"]
        dist.all_gather_object(gathered, {"path": c.get("path"),
                                          "value": c["value"].cpu().numpy() if c else None})
        if rank == 0:
            other = gathered[world - 1]
            ex0 = qf.PlanExecutor(base.fix_outputs(units[0][1]), plan)
            t = ex0.run(other["path"])
            t = t.transpose_to(order) if order else t
            mine = t.data[:width].cpu().numpy()
            err = float(np.linalg.norm(mine - other["value"]) / max(np.linalg.norm(mine), 1e-300))
            selfcheck = {"what": f"rank {world - 1}'s path {other['path']} of unit 0 recomputed "
                                 f"on rank 0 (N=1)", "rel_l2": err, "ok": err < 1e-4}
            if err >= 1e-4:
                raise AssertionError(f"N>1 self-check failed: {selfcheck}")
        barrier(world)

    # ---- end to end through the public API (host in, host out); the timed
    # walk's cached intermediates (up to ~70 GiB at config 4) are released
    # first so the API call has the device to itself
    unit_results = [[[float(v.real), float(v.imag)] for v in r[:4].cpu().numpy()]
                    for r in state["results"][:4]]
    state.update(ex=None, acc=None, results=[], contrib={})
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    h2d = d2h = 0
    e2e_s = []
    for u in range(max(0, args.e2e_units)):
        bits, fixed = units[u]
        e_eng = qf.AmplitudeEngine(circ, plan, device=local, group=group)
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if c_sites:
            s_ab = "".join(str(fixed.get(q, 0)) for q in range(circ.n))
            res = e_eng.amplitude_batch(0, s_ab, c_sites, width, seed=SEED, fidelity=fid)
            d2h = width * 8
        else:
            res = e_eng.amplitude(0, bits, fid)
            d2h = 8
        e1.record()
        torch.cuda.synchronize()
        e2e_s.append(max(time.perf_counter() - t0, e0.elapsed_time(e1) / 1e3))
        h2d = sum(arr.nbytes for stack in qf.build_3d(circ, 0, None).blocks.values()
                  for _, arr in stack)
        del e_eng
    e2e_unit_s = max_over_ranks(float(np.mean(e2e_s)) if e2e_s else float("nan"), world, dev)
    e2e = wl["amps_per_unit"] / e2e_unit_s

    result = None
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_projection(args.workload, host_cores(), args.cpu_seconds)
        result = {
            "metric": "amplitudes/s", "value": round(value, 6), "unit": "amplitudes/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 2), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c64 (fp32 complex; 3xTF32 on tcgen05 tensor cores)",
            "data": "synthetic (seeded RQC + seeded bit-strings; the paper's circuit files are "
                    "not in the container)",
            "config": {"workload": wl["desc"], "lattice": wl["lattice"], "depth": wl["depth"],
                       "circuit_seed": SEED, "fidelity": wl["f"], "paths_per_unit": n_paths,
                       "amplitudes_per_unit": wl["amps_per_unit"],
                       "step": "one contraction path per rank (PlanExecutor.run)",
                       "parallelism": f"slices (paths) sharded x{world}, one all-reduce per unit",
                       "l2": "inputs larger than L2 (operands up to 8 GiB)"},
            "flops_per_unit_reference_convention": int(flops_unit),
            "executed_flops_per_step": int(exec_flops / args.steps),
            "executed_tflops": round(exec_flops / args.steps / (ms / 1e3) / 1e12, 2),
            "reference_equivalent_tflops": round(paths_per_s / n_paths * flops_unit / 1e12, 2),
            "gemm_mode": qf.get_gemm_mode(),
            "e2e": {"value": round(e2e, 6) if e2e_s else None, "unit": "amplitudes/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "seconds_per_unit": round(e2e_unit_s, 2) if e2e_s else None,
                    "api": ("AmplitudeEngine(circuit, plan).amplitude_batch(0, s_ab, c_sites, 64)"
                            if c_sites else "AmplitudeEngine(circuit, plan).amplitude(0, bits, f)")
                           + " per unit, network built from the host circuit every call"},
            "roofline": roof,
            "kernels": {k: {"launches": x["launches"], "ms_per_step": round(x["ms"] / args.steps, 2),
                            "share": round(x["ms"] / max(step_kernel_ms, 1e-9), 4)}
                        for k, x in sorted(kerns.items(), key=lambda kv: -kv[1]["ms"])[:8]},
            "gpu_launches": int(launches // max(args.steps, 1)),
            "clocks": clocks.summary(), "cpu_baseline": cpu, "self_check": selfcheck,
            "units_completed_in_run": state["u"],
            # amplitudes of the units completed inside this run (first 4 values each)
            "unit_results": unit_results,
        }
        # issued TF32 MMA flops / (2048 MACs/clk/SM x 148 SMs x the SM clock
        # measured under load): what the tensor pipe did at the clock it ran at
        mhz = (result["clocks"] or {}).get("sm_mhz")
        if mhz:
            pipe = 2048 * 2 * sm_count_of(torch) * mhz * 1e6 / 1e12
            roof["tensor_pipe_util_at_measured_clock"] = round(
                roof["achieved"] * 2 * tc.tc3_real_macs_per_complex_mac(roof["kernel"]) / 8 / pipe, 4)
    return result


def _cpu_unit_worker(args):
    """One unit (amplitude / open batch) of the oracle port at reduced depth."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    workload, idx = args
    import paper_1811_09599_b200 as qf
    from oracle import rqc_oracle
    wl = PATH_WORKLOADS[workload]
    lat = qf.Lattice.named(wl["lattice"])
    circ = qf.generate_rqc(lat, wl["cpu_depth"], SEED)
    plan = qf.load_plan(wl["plan"])
    units, c_sites = path_units(wl, circ, plan, idx + 1)
    bits, fixed = units[idx]
    eng = rqc_oracle.OracleEngine(qf.write_circuit(circ), qf.format_plan(plan), np.complex64)
    t0 = time.perf_counter()
    if c_sites:
        s_ab = "".join(str(fixed.get(q, 0)) for q in range(circ.n))
        _, _, flops, _ = eng.amplitude_batch(0, s_ab, c_sites, 2 ** len(c_sites), seed=SEED,
                                             f=wl["f"], fseed=SEED)
    else:
        _, _, _, flops = eng.amplitude(0, bits, wl["f"], SEED)
    return time.perf_counter() - t0, flops


def cpu_projection(workload: str, procs: int, seconds: float) -> dict:
    """The oracle port (the reference algorithm in numpy) on the host cores at
    a reduced depth where one unit takes ~a second, same plan and fidelity,
    `procs` single-threaded processes each walking whole units for about
    `seconds`; its sustained GFLOP/s (reference convention) divided by the
    full-depth flops per unit is the PROJECTED CPU rate (full depth is
    infeasible on CPU: ~days per config-4 amplitude)."""
    import multiprocessing as mp
    import paper_1811_09599_b200 as qf
    from paper_1811_09599_b200 import plan_tools as pt
    wl = PATH_WORKLOADS[workload]
    env_keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in env_keys}
    for k in env_keys:
        os.environ[k] = "1"
    try:
        ctx = mp.get_context("spawn")
        with ctx.Pool(procs) as pool:
            first = pool.map(_cpu_unit_worker, [(workload, i) for i in range(procs)])  # warm
            per = max(t for t, _ in first)
            rounds = max(1, int(seconds / max(per, 1e-3)))
            t0 = time.perf_counter()
            out = pool.map(_cpu_unit_worker, [(workload, i % 64) for i in range(procs * rounds)])
            wall = time.perf_counter() - t0
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    flops = sum(f for _, f in out)
    gfs = flops / wall / 1e9
    lat = qf.Lattice.named(wl["lattice"])
    plan = qf.load_plan(wl["plan"])
    c_sites = tuple(sorted(plan.batch_sites[:wl["open"]])) if wl["open"] else ()
    full = pt.fidelity_flops(plan, lat, wl["depth"], wl["f"], SEED, open_sites=c_sites)
    rate = gfs * 1e9 / full * wl["amps_per_unit"]
    return {"value": rate, "unit": "amplitudes/s", "cores": procs, "kind": "port",
            "projection": True, "seconds": round(wall, 2), "gflops": round(gfs, 2),
            "sample": f"{len(out)} units of {workload} at depth {wl['cpu_depth']} (same plan, "
                      f"f={wl['f']}) through oracle/rqc_oracle.py (numpy restatement of the "
                      f"reference), {procs} processes x 1 thread; measured {gfs:.1f} GFLOP/s "
                      f"(reference flop convention) / {full:.3e} flops per unit at "
                      f"{wl['depth']} = projected full-depth rate"}


def run_reference(args):
    """The reference algorithm on the host cores (the oracle port, all
    cores), same metric and config as the GPU arm; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    sys.path.insert(0, ROOT)
    import paper_1811_09599_b200 as qf  # host-side circuit/plan text only
    if args.workload in PATH_WORKLOADS:
        wl = PATH_WORKLOADS[args.workload]
        rates = [cpu_projection(args.workload, host_cores(), args.cpu_seconds)
                 for _ in range(args.warmup + args.steps)][args.warmup:]
        secs = sum(r["seconds"] for r in rates)
        gfs = float(np.mean([r["gflops"] for r in rates]))
        value = float(np.mean([r["value"] for r in rates]))
        cpu = dict(rates[-1])
        cpu["value"] = value
        return {"impl": "reference", "metric": "amplitudes/s", "value": value,
                "unit": "amplitudes/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(secs / len(rates) * 1e3, 2),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c64",
                "data": "synthetic (seeded RQC + seeded bit-strings)",
                "config": {"workload": wl["desc"], "lattice": wl["lattice"],
                           "depth": wl["depth"], "fidelity": wl["f"],
                           "measured_at_depth": wl["cpu_depth"],
                           "projection": "full depth is infeasible on CPU: GFLOP/s measured on the "
                                         "same plan at reduced depth / full-depth flops per unit"},
                "cpu_baseline": cpu, "gflops": round(gfs, 2),
                "e2e": {"value": value, "unit": "amplitudes/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
    wl = args.workload if args.workload in WORKLOADS else "config2"
    LATTICE, DEPTH, N_CUTS, N_BITSTRINGS = WORKLOADS[wl][:4]
    lat = qf.Lattice.named(LATTICE)
    circ = qf.generate_rqc(lat, DEPTH, SEED)
    plan = qf.grid_plan(lat, n_cuts=N_CUTS)
    outs = bitstrings(0, circ.n, N_BITSTRINGS)
    cores = host_cores()
    sample = max(cores, min(N_BITSTRINGS, int(args.cpu_sample)))
    rates = []
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_rate(qf.write_circuit(circ), qf.format_plan(plan), outs[:sample], cores,
                            f"the {N_BITSTRINGS} {wl} bit-strings")
        if i >= args.warmup:
            rates.append(r)
    secs = sum(r["seconds"] for r in rates)
    value = sample * len(rates) / secs
    cpu = dict(rates[-1])
    cpu["value"] = round(value, 3)
    return {"impl": "reference", "metric": "amplitudes/s", "value": round(value, 3),
            "unit": "amplitudes/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(secs / len(rates) * 1e3, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c64",
            "data": "synthetic (seeded RQC + seeded bit-strings)",
            "config": workload_config("bitstrings", 1, wl),
            "cpu_baseline": cpu,
            "e2e": {"value": round(value, 3), "unit": "amplitudes/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def _compact(r: dict) -> dict:
    out = {"workload": r["config"]["workload"], "value": r["value"], "unit": r["unit"],
           "ms_per_step": r.get("ms_per_step"), "steps": r.get("steps"),
           "e2e": (r.get("e2e") or {}).get("value"),
           "roofline": {k: r["roofline"].get(k) for k in ("bound", "kernel", "achieved", "peak",
                                                            "unit", "frac")},
           "gpu_launches": r.get("gpu_launches"), "self_check": r.get("self_check")}
    for k in ("per_size", "executed_tflops", "units_completed_in_run", "single_call"):
        if k in r:
            out[k] = r[k]
    e2e = r.get("e2e") or {}
    if e2e.get("seconds_per_unit"):
        out["e2e_seconds_per_unit"] = e2e["seconds_per_unit"]
    cpu = r.get("cpu_baseline")
    if cpu:
        out["cpu_baseline"] = {k: cpu.get(k) for k in ("value", "unit", "cores", "kind", "projection",
                                                       "gflops", "seconds")}
    return out


def secondary_workloads(args) -> list:
    """The other BASELINE configs measured in the same run, summarised beside
    the headline (short runs: config 2 = configs[1], the batched bit-string
    workload; config 1; config 3 = 8 of the 64 seeded permutations per size;
    config 5 = path steps of the first open-qubit batch)."""
    import torch
    runs = (("config2", run_gpu, {"steps": 10}),
            ("config1", run_gpu, {"steps": 10}),
            ("permute", run_permute, {"steps": 3, "perms": 8}),
            # config 5: 10 path steps, ONE whole 64-amplitude batch (328 paths)
            # through amplitude_batch() as its e2e, and a short CPU projection
            ("config5", run_paths, {"steps": 10, "e2e_units": 1, "no_cpu_baseline": False,
                                    "cpu_seconds": 6.0}))
    want = [w.strip() for w in str(args.secondary_workloads).split(",") if w.strip()]
    out = []
    for name, fn, over in runs:
        if name not in want or name == args.workload:
            continue
        sub = argparse.Namespace(**vars(args))
        sub.workload, sub.warmup, sub.no_cpu_baseline = name, 3, True
        for k, v in over.items():
            setattr(sub, k, v)
        if args.no_cpu_baseline:
            sub.no_cpu_baseline = True
        try:
            r = fn(sub)
            if r is not None:
                out.append(_compact(r))
        except Exception as exc:  # the headline stands on its own
            out.append({"workload": name, "error": repr(exc)[:300]})
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--shard", choices=["bitstrings", "slices"], default="bitstrings",
                    help="config1/config2 only: bit-strings per rank (no collective) or the "
                         "slices of one batch split over the ranks (one all-reduce)")
    ap.add_argument("--gemm", choices=["auto", "ffma", "tc3"], default=None)
    ap.add_argument("--tc3-variant", type=int, default=0,
                    help="pin a tensor-core kernel flavour (qf_tc3_set_variant) for A/B runs")
    ap.add_argument("--cpu-sample", type=int, default=1024,
                    help="config1/2: bit-strings timed on the host cores")
    ap.add_argument("--cpu-seconds", type=float, default=15.0,
                    help="config4/5: seconds of oracle work per CPU-projection sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=["config4", "config4f1", "config5", "config2", "config1", "permute"],
                    default="config4",
                    help="config4 = headline (the largest single-GPU config, tensor-core bound); "
                         "config5; config2 (BASELINE configs[1]); config1; permute = config 3")
    ap.add_argument("--secondary", type=int, default=1,
                    help="config4/5: also run short measurements of the other configs "
                         "(reported under 'secondary')")
    ap.add_argument("--secondary-workloads", default="config2,config1,permute,config5")
    ap.add_argument("--e2e-units", type=int, default=1,
                    help="config4/5: whole units (amplitudes / batches) timed through the API")
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="launch the plan walk eagerly instead of replaying a captured CUDA graph")
    ap.add_argument("--no-late", dest="late", action="store_false",
                    help="slice every output up front (no late output slicing)")
    ap.add_argument("--perm-sizes", default="24,28,30")
    ap.add_argument("--perms", type=int, default=64)
    ap.add_argument("--perm-graph", type=int, default=1,
                    help="time the K permutes of a case as one CUDA-graph replay (1) or eagerly (0)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        out = run_reference(args)
    else:
        import torch
        rank, world, local = dist_env()
        torch.cuda.set_device(local)
        init_dist(world, "nccl")
        if args.tc3_variant:
            from paper_1811_09599_b200 import _lib
            _lib.load().qf_tc3_set_variant(args.tc3_variant)
        try:
            if args.workload == "permute":
                out = run_permute(args)
            elif args.workload in PATH_WORKLOADS:
                out = run_paths(args)
                if args.secondary:
                    sec = secondary_workloads(args)
                    if out is not None:
                        out["secondary"] = sec
            else:
                out = run_gpu(args)
        finally:
            if world > 1:
                import torch.distributed as dist
                dist.barrier()
                dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
