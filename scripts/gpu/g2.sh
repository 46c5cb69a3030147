mkdir -p gpurun_out
for v in 0 26 27; do
for s in 8192,8192,8192 32768,32768,32768 4096,4096,65536; do
  timeout 300 python scripts/gemm_probe.py --shape $s --seconds 5 --variant $v >> gpurun_out/g2_probe.jsonl 2>>gpurun_out/g2_err.txt
done
done
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_gemm.py -x -q > gpurun_out/g2_tests.txt 2>&1
echo done
