#!/bin/bash
# wide Gauss kernel: correctness (short timeouts: a hang must not eat the budget), then A/B probes
mkdir -p gpurun_out
rm -f gpurun_out/wide_probe.jsonl
timeout 60 python scripts/gemm_probe.py --shape 256,256,1024 --seconds 0.05 --variant 40 --check 1 > gpurun_out/wide_first.txt 2>&1
echo "first rc=$?" >> gpurun_out/wide_first.txt
cat gpurun_out/wide_first.txt
grep -q "first rc=0" gpurun_out/wide_first.txt || exit 1
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "wide" --timeout 60 > gpurun_out/wide_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/wide_tests.txt
tail -5 gpurun_out/wide_tests.txt
for shape in 8192,8192,8192 4096,4096,65536 1048576,1024,1024 32768,32768,32768; do
  for v in 40 41; do
    timeout 120 python scripts/gemm_probe.py --shape $shape --seconds 3 --variant $v --check 1 >> gpurun_out/wide_probe.jsonl 2>&1
  done
done
cat gpurun_out/wide_probe.jsonl
