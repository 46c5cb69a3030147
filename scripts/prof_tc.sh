# ncu full captures of the WS tensor-core GEMM: config-2's gathered shape
# (inside the bench step) and a large square GEMM.  usage: prof_tc.sh <tag>
mkdir -p gpurun_out
T=${1:-tc}
bash scripts/profile.sh ${T}_c2 tc3w 10
CMD="python scripts/gemm_one.py 1 8192 8192 8192 2 0 2"
$CMD && ncu --set full --clock-control none --import-source on -k regex:tc3w -s 1 -c 1 -o gpurun_out/${T}_8192 $CMD > gpurun_out/${T}_8192_ncu.log 2>&1; echo ncu_rc=$?
