mkdir -p gpurun_out
CMD="python scripts/gemm_one.py 1 4096 4096 4096 2 0 3"
$CMD && ncu --set full --clock-control none --import-source on -k regex:tc3s -s 1 -c 1 -o gpurun_out/tc3s_v4_4096 $CMD > gpurun_out/tc3s_ncu.log 2>&1; echo ncu_rc=$?
python bench.py --steps 10 --warmup 3 --no-cpu-baseline | cut -c 1-400
python scripts/step_profile.py auto 1024 | head -14
