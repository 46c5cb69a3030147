mkdir -p gpurun_out
for d in 44 47; do
  QF_TC3_DEBUG=$d timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 2 --check 0 | sed "s/^/dbg=$d /" >> gpurun_out/g23_probe.txt 2>&1
done
for v in 19; do
  QF_TC3_DEBUG=44 timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 2 --check 0 --variant $v | sed "s/^/dbg=44 v19 /" >> gpurun_out/g23_probe.txt 2>&1
done
echo done
