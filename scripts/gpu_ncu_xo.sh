mkdir -p gpurun_out
python scripts/ncu_c2_step.py > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tc3k" -c 12 -o gpurun_out/r1k_tc python scripts/ncu_c2_step.py > gpurun_out/ncu_k.log 2>&1; echo rc=$?
