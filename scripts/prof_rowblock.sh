# ncu full captures of the row-block GEMM at config-2 shapes
mkdir -p gpurun_out
T=${1:-rb}
CMD1="python scripts/contract_one.py '@b a b c k d e' '@b k n' 8 3"
CMD2="python scripts/gemm_one.py 1024 4096 8 64 1 0 3"
eval $CMD1 && eval ncu --set full --clock-control none --import-source on -k regex:rowblock -s 1 -c 1 -o gpurun_out/${T}_m32768 $CMD1 > gpurun_out/${T}_1.log 2>&1; echo ncu_rc=$?
$CMD2 && ncu --set full --clock-control none --import-source on -k regex:rowblock -s 1 -c 1 -o gpurun_out/${T}_n8k64 $CMD2 > gpurun_out/${T}_2.log 2>&1; echo ncu_rc=$?
