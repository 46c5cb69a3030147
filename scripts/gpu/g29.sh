mkdir -p gpurun_out
for d in 44 108; do
  QF_TC3_DEBUG=$d timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 2 --check 0 | sed "s/^/dbg=$d /" >> gpurun_out/g29_probe.txt 2>&1
done
echo done
