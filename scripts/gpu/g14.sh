mkdir -p gpurun_out
for v in 0 34; do for d in 0 3; do
  QF_TC3_DEBUG=$d timeout 300 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 2 --check 0 --variant $v | sed "s/^/dbg=$d /" >> gpurun_out/g14_probe.txt 2>&1
done; done
echo done
