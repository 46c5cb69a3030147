mkdir -p gpurun_out
CMD="python scripts/gemm_one.py 1 4096 4096 4096 2 0 3"
$CMD && ncu --set full --clock-control none --import-source on -k regex:tc3s -s 1 -c 1 -o gpurun_out/tc3s_4096 $CMD > gpurun_out/tc3s_ncu.log 2>&1; echo ncu_rc=$?
CMD2="python scripts/gemm_one.py 1 4096 4096 4096 2 2 3"
$CMD2 && ncu --set full --clock-control none --import-source on -k regex:tc3_kernel -s 1 -c 1 -o gpurun_out/tc3v1_4096 $CMD2 > gpurun_out/tc3v1_ncu.log 2>&1; echo ncu2_rc=$?
