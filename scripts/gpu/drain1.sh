#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/drain_probe.jsonl
timeout 60 python scripts/gemm_probe.py --shape 1024,256,1024 --seconds 0.05 --variant 46 --check 1 > gpurun_out/drain_first.txt 2>&1
echo "first rc=$?" >> gpurun_out/drain_first.txt; cat gpurun_out/drain_first.txt
grep -q "first rc=0" gpurun_out/drain_first.txt || exit 1
for rep in 1 2; do
for shape in 8192,8192,8192 32768,32768,32768 1048576,256,256; do
  for v in 43 46 44; do
    timeout 120 python scripts/gemm_probe.py --shape $shape --seconds 3 --variant $v --check 1 >> gpurun_out/drain_probe.jsonl 2>&1
  done
done
done
python - <<'PY'
import json
for l in open("gpurun_out/drain_probe.jsonl"):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d["shape"], d["variant"], d["burst_tflops"], d["sustained_tflops"], d["sm_mhz_median"], d.get("rel_l2_vs_f64"))
PY
