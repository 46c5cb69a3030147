"""Summarise ncu outputs for profiles/: per-kernel launch shares from a
`--metrics gpu__time_duration.sum --csv` log, and key metrics of a
`--set full` report (read with `ncu -i ... --page raw --csv`)."""
import csv, io, subprocess, sys
from collections import defaultdict


def launches(path):
    rows = [l for l in open(path) if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(rows)))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:90]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1e3 if unit == "ns" else v * (1e3 if unit == "ms" else 1.0)  # -> us
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values()) or 1
    out = [f"{'kernel':90s} {'launches':>8s} {'total_us':>12s} {'share':>7s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:90s} {n:8d} {t:12.1f} {t / tot:7.3f}")
    out.append(f"{'TOTAL':90s} {sum(v[0] for v in agg.values()):8d} {tot:12.1f}")
    return "\n".join(out)


KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__t_bytes.sum", "lts__t_bytes.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rd = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rd[0], rd[1], rd[2:]
    out = []
    for row in vals:
        for k in KEYS:
            for i, h in enumerate(hdr):
                if h == k or (k.endswith("tensor_cycles_active.avg.pct_of_peak_sustained_active") and h.startswith("sm__pipe_tensor") and "pct" in h):
                    out.append(f"{h} [{units[i]}] = {row[i]}")
                    break
        out.append("")
    return "\n".join(out)


def family(kernel_name):
    """'void tc::cgemm_tc3k_kernel<8, 4>(GemmArgs, ...)' -> 'cgemm_tc3k' (the
    names bench.py's per-kernel table uses)."""
    name = kernel_name.split("(")[0].split("<")[0].replace("void ", "").strip()
    name = name.split("::")[-1]
    return name[:-len("_kernel")] if name.endswith("_kernel") else name


def traffic(path):
    """Per kernel family of a `--metrics gpu__time_duration.sum,dram__bytes_read.sum,
    dram__bytes_write.sum --csv` capture: launches, DRAM bytes, time (JSON)."""
    import json
    rows = [l for l in open(path) if l.startswith('"')]
    agg = defaultdict(lambda: {"ids": set(), "dram_read": 0.0, "dram_write": 0.0, "ns": 0.0})
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3,
             "usecond": 1e3, "nsecond": 1, "ms": 1e6, "msecond": 1e6}
    for r in csv.DictReader(io.StringIO("".join(rows))):
        a = agg[family(r["Kernel Name"])]
        a["ids"].add(r["ID"])
        v = float(r["Metric Value"].replace(",", "")) * scale.get(r["Metric Unit"], 1)
        key = {"dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
               "gpu__time_duration.sum": "ns"}.get(r["Metric Name"])
        if key:
            a[key] += v
    out = {}
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["ns"]):
        n = len(a["ids"])
        out[k] = {"launches": n, "dram_bytes_per_launch": round((a["dram_read"] + a["dram_write"]) / n),
                  "dram_read": round(a["dram_read"]), "dram_write": round(a["dram_write"]),
                  "us": round(a["ns"] / 1e3, 1)}
    return json.dumps(out, indent=1)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print({"launches": launches, "full": full, "traffic": traffic}[kind](path))
