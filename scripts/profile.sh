#!/bin/bash
# ncu evidence for profiles/: launch list of one bench run + one full capture
# of the top kernel.  Each ncu pass follows a plain run of the same command.
# usage: bash scripts/profile.sh <tag> <kernel-regex> <skip> [bench args...]
set -u
mkdir -p gpurun_out
TAG=$1; KRE=$2; SKIP=$3; shift 3
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline $*"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1
echo "launch-list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:${KRE} -s ${SKIP} -c 1 \
    -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "full rc=$?"
