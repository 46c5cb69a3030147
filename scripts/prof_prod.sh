mkdir -p gpurun_out
QF_TC3_VARIANT=17 python scripts/step_profile.py auto 1024 2>/dev/null | head -3
CMD="python scripts/gemm_one.py 1 4096 4096 4096 2 18 2"
$CMD && ncu --set full --clock-control none --import-source on -k regex:tc3k -s 1 -c 1 -o gpurun_out/prod_4096 $CMD > gpurun_out/prod.log 2>&1; echo ncu_rc=$?
