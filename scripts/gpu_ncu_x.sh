mkdir -p gpurun_out
QF_TC3_VARIANT=26 python scripts/ncu_c2_step.py > /dev/null 2>&1
QF_TC3_VARIANT=26 timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tc3k" -c 8 -o gpurun_out/r1j_x python scripts/ncu_c2_step.py > gpurun_out/ncu_x.log 2>&1; echo rc=$?
