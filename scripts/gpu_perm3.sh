mkdir -p gpurun_out
QF_PERM_DEBUG=1 python scripts/perm_one.py 28 > gpurun_out/perm28.txt 2>&1
QF_PERM_DEBUG=1 python scripts/perm_one.py 24 > gpurun_out/perm24.txt 2>&1
python scripts/perm_one.py 28 0 2 && ncu --set full --clock-control none --import-source on -k regex:permute -s 3 -c 1 -o gpurun_out/perm28_c0 python scripts/perm_one.py 28 0 1 > gpurun_out/ncu_perm.log 2>&1; echo ncu=$?
