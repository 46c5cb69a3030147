mkdir -p gpurun_out
for v in 0 19; do
for s in 8192,8192,8192 32768,32768,32768; do
  timeout 300 python scripts/gemm_probe.py --shape $s --seconds 5 --variant $v >> gpurun_out/g7_probe.jsonl 2>>gpurun_out/g7_err.txt
done
done
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -k "tcgen05" > gpurun_out/g7_tests.txt 2>&1
timeout 300 python scripts/single_call.py > gpurun_out/g7_single.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_acceptance.py -q > gpurun_out/g7_acc.txt 2>&1
timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/g7_plain.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cgemm_tc3 -s 1 -c 1 -o gpurun_out/g7_tc3g_8192 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/g7_ncu.log 2>&1
echo done
