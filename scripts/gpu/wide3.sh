#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/pair_probe.jsonl
timeout 60 python scripts/gemm_probe.py --shape 1024,256,1024 --seconds 0.05 --variant 43 --check 1 > gpurun_out/pair_first.txt 2>&1
echo "first rc=$?" >> gpurun_out/pair_first.txt
cat gpurun_out/pair_first.txt
grep -q "first rc=0" gpurun_out/pair_first.txt || exit 1
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "wide" --timeout 60 > gpurun_out/pair_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/pair_tests.txt
tail -5 gpurun_out/pair_tests.txt
for shape in 8192,8192,8192 4096,4096,65536 1048576,1024,1024 32768,32768,32768; do
  for v in 40 43; do
    timeout 120 python scripts/gemm_probe.py --shape $shape --seconds 3 --variant $v --check 1 >> gpurun_out/pair_probe.jsonl 2>&1
  done
done
cat gpurun_out/pair_probe.jsonl
