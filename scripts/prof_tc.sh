mkdir -p gpurun_out
CMD="python scripts/gemm_one.py 1024 4096 64 64 2 0 3"
$CMD && ncu --set full --clock-control none --import-source on -k regex:tc3w -s 1 -c 1 -o gpurun_out/tc3w_c2shape $CMD > gpurun_out/tc3w_c2_ncu.log 2>&1; echo ncu_rc=$?
CMD="python scripts/gemm_one.py 1 8192 8192 8192 2 0 2"
$CMD && ncu --set full --clock-control none --import-source on -k regex:tc3w -s 1 -c 1 -o gpurun_out/tc3w_8192 $CMD > gpurun_out/tc3w_8192_ncu.log 2>&1; echo ncu_rc=$?
