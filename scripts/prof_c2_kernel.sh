# ncu full captures of one kernel family inside a config-2 step
# usage: prof_c2_kernel.sh <tag> <kernel-regex> <skip> <count>
mkdir -p gpurun_out
T=$1; KRE=$2; SKIP=$3; CNT=$4
CMD="python scripts/step_profile.py auto 1024"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c $CNT -o gpurun_out/${T} $CMD > gpurun_out/${T}.log 2>&1; echo ncu_rc=$?
