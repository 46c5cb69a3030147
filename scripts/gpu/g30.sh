mkdir -p gpurun_out
QF_TC3_DEBUG=44 timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/g30_plain.txt 2>&1 && \
QF_TC3_DEBUG=44 timeout 600 ncu --set full --import-source on --clock-control none -k regex:cgemm_tc3 -s 1 -c 1 -o gpurun_out/g30_dbg44 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/g30_ncu.log 2>&1
echo done
