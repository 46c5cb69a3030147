# ncu full captures of the long-K TC kernels (tc3w vs TMEM-master tc3k) at 8192^3 and 4096^3
mkdir -p gpurun_out
T=${1:-lk}
for v in 0 13; do
  for n in 4096 8192; do
    CMD="python scripts/gemm_one.py 1 $n $n $n 2 $v 2"
    $CMD && ncu --set full --clock-control none --import-source on -k regex:"tc3w|tc3k" -s 1 -c 1 -o gpurun_out/${T}_v${v}_$n $CMD > gpurun_out/${T}_v${v}_$n.log 2>&1; echo ncu_rc=$?
  done
done
