mkdir -p gpurun_out
for e in 2 3; do python scripts/contract_one.py '@b a k1 b c d k2' '@b k1 k2 n' 8 3 $e; python scripts/contract_one.py '@b a b c k d e' '@b k n' 8 3 $e; python scripts/contract_one.py '@b a b c d k1 k2' '@b k1 k2 n' 8 3 $e; done
CMD="python scripts/contract_one.py '@b a k1 b c d k2' '@b k1 k2 n' 8 3 3"
eval ncu --set full --clock-control none --import-source on -k regex:rowstream -s 1 -c 1 -o gpurun_out/rs2_gk $CMD > gpurun_out/rs2.log 2>&1; echo ncu_rc=$?
