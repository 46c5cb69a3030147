mkdir -p gpurun_out
for d in 8 11 15; do
  QF_TC3_DEBUG=$d timeout 300 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 2 --check 0 | sed "s/^/dbg=$d /" >> gpurun_out/g15_probe.txt 2>&1
done
echo done
