"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r)
hdr = rows[hdr_i]
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
data = [r for r in rows[hdr_i + 1:] if len(r) > si]
tot = sum(float(r[si] or 0) for r in data) or 1
for r in sorted(data, key=lambda r: -float(r[si] or 0))[:top]:
    print(f"{float(r[si]) / tot:6.3f}  {r[src].strip()[:90]}")
