mkdir -p gpurun_out
for e in 2 3; do python scripts/contract_one.py '@b k1 a k2 b c d' '@b k1 k2 n' 8 3 $e; done
CMD="python scripts/contract_one.py '@b k1 a k2 b c d' '@b k1 k2 n' 8 3 3"
eval ncu --set full --clock-control none --import-source on -k regex:rowstream -s 1 -c 1 -o gpurun_out/rs3_rc $CMD > gpurun_out/rs3.log 2>&1; echo ncu_rc=$?
