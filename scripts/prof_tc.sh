mkdir -p gpurun_out
CMD="python scripts/gemm_one.py 1 4096 4096 4096 2 6 3"
$CMD && ncu --set full --clock-control none --import-source on -k regex:tc3pair -s 1 -c 1 -o gpurun_out/tc3pair_4096 $CMD > gpurun_out/tc3pair_ncu.log 2>&1; echo ncu_rc=$?
