set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/g1_smi.txt
for s in 4096,4096,4096 8192,8192,8192 16384,16384,16384 32768,32768,32768 4096,4096,65536; do
  timeout 300 python scripts/gemm_probe.py --shape $s --seconds 6 --cublas 0 >> gpurun_out/g1_probe.jsonl 2>>gpurun_out/g1_err.txt
done
timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 1 --cublas 1 >> gpurun_out/g1_probe.jsonl 2>>gpurun_out/g1_err.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cgemm_tc3k -s 1 -c 1 -o gpurun_out/g1_tc3k_8192 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/g1_ncu.log 2>&1
echo done
