mkdir -p gpurun_out
T=${1:-lk3}
for n in 8192; do
  CMD="python scripts/gemm_one.py 1 $n $n $n 2 0 2"
  $CMD && ncu --set full --clock-control none --import-source on -k regex:"tc3k" -s 1 -c 1 -o gpurun_out/${T}_$n $CMD > gpurun_out/${T}_$n.log 2>&1; echo ncu_rc=$?
done
