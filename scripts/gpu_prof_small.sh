mkdir -p gpurun_out
python scripts/ncu_c2_step.py > /dev/null 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"rowblock|rowstream" -c 4 -o gpurun_out/r1e_rs python scripts/ncu_c2_step.py > gpurun_out/ncu_rs.log 2>&1; echo rc=$?
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tc3k" -c 17 -o gpurun_out/r1e_tc python scripts/ncu_c2_step.py > gpurun_out/ncu_tc.log 2>&1; echo rc=$?
