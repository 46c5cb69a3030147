mkdir -p gpurun_out
CMD="python scripts/gemm_one.py 1 4096 4096 4096 2 0 3"
$CMD && ncu --set full --clock-control none --import-source on -k regex:tc3w -s 1 -c 1 -o gpurun_out/tc3w_4096 $CMD > gpurun_out/tc3w_ncu.log 2>&1; echo ncu_rc=$?
