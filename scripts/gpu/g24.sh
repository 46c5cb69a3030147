mkdir -p gpurun_out
for v in 0 30 31; do
  QF_TC3_DEBUG=44 timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 2 --check 0 --variant $v | sed "s/^/dbg=44 /" >> gpurun_out/g24_probe.txt 2>&1
done
timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 3 --check 0 | sed "s/^/dbg=0 /" >> gpurun_out/g24_probe.txt 2>&1
echo done
