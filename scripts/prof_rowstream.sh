mkdir -p gpurun_out
T=${1:-rs}
CMD2="python scripts/gemm_one.py 1024 4096 8 64 1 0 3"
$CMD2 && ncu --set full --clock-control none --import-source on -k regex:rowstream -s 1 -c 1 -o gpurun_out/${T}_n8k64 $CMD2 > gpurun_out/${T}_2.log 2>&1; echo ncu_rc=$?
