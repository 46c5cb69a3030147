mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -k "tcgen05" > gpurun_out/g11_tests.txt 2>&1
for v in 0 19; do
for s in 8192,8192,8192 32768,32768,32768 4096,4096,65536; do
  timeout 300 python scripts/gemm_probe.py --shape $s --seconds 5 --variant $v >> gpurun_out/g11_probe.jsonl 2>>gpurun_out/g11_err.txt
done
done
timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/g11_plain.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cgemm_tc3 -s 1 -c 1 -o gpurun_out/g11_tc3g_8192 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/g11_ncu.log 2>&1
echo done
