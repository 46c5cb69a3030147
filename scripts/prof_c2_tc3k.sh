# ncu full captures of the short-K TC launches of one config-2 step
mkdir -p gpurun_out
T=${1:-c2k}
CMD="python scripts/step_profile.py auto 1024"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:tc3k -s 21 -c 7 -o gpurun_out/${T} $CMD > gpurun_out/${T}.log 2>&1; echo ncu_rc=$?
