mkdir -p gpurun_out
for v in 30 31 32; do
for s in 8192,8192,8192 32768,32768,32768 4096,4096,65536; do
  timeout 300 python scripts/gemm_probe.py --shape $s --seconds 5 --variant $v >> gpurun_out/g4_probe.jsonl 2>>gpurun_out/g4_err.txt
done
done
timeout 1200 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/g4_bench.json 2> gpurun_out/g4_bench.err
echo done
