mkdir -p gpurun_out
for v in 34 0; do
  QF_TC3_DEBUG=44 timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 2 --check 0 --variant $v | sed "s/^/dbg=44 /" >> gpurun_out/g26_probe.txt 2>&1
  QF_TC3_DEBUG=3 timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 2 --check 0 --variant $v | sed "s/^/dbg=3 /" >> gpurun_out/g26_probe.txt 2>&1
done
echo done
