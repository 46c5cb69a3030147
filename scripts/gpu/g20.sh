mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -k "tcgen05" > gpurun_out/g20_tests.txt 2>&1
for v in 0 34; do
for s in 8192,8192,8192 32768,32768,32768 4096,4096,65536; do
  timeout 300 python scripts/gemm_probe.py --shape $s --seconds 5 --variant $v >> gpurun_out/g20_probe.jsonl 2>>gpurun_out/g20_err.txt
done
done
QF_TC3_DEBUG=3 timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 2 --check 0 >> gpurun_out/g20_probe.jsonl 2>&1
echo done
