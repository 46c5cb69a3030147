# ncu --set full of the narrow-N CUDA-core GEMMs of one config-2 step
mkdir -p gpurun_out
python scripts/ncu_c2_step.py > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"rowblock|rowstream" -c 6 -o gpurun_out/r1g_narrow python scripts/ncu_c2_step.py > gpurun_out/ncu_narrow.log 2>&1; echo rc=$?
