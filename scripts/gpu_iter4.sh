mkdir -p gpurun_out
QF_TC3_VARIANT=22 QF_ORDER=1 python scripts/step_profile.py auto 1024 > gpurun_out/iter_prof22.txt 2>&1
python scripts/ncu_c2_step.py > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tc3k" -c 20 -o gpurun_out/r1g_tc2 python scripts/ncu_c2_step.py > gpurun_out/ncu_tc.log 2>&1; echo rc=$?
