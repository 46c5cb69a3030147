# ncu full captures of the short-K tensor-core kernel at config-2 shapes.
# usage: prof_short.sh <tag>
mkdir -p gpurun_out
T=${1:-sk}
for shp in "1024 4096 64 8" "1024 4096 64 64"; do
  n=$(echo $shp | tr ' ' _)
  CMD="python scripts/gemm_one.py $shp 2 0 3"
  $CMD && ncu --set full --clock-control none --import-source on -k regex:tc3k -s 1 -c 1 -o gpurun_out/${T}_$n $CMD > gpurun_out/${T}_$n.log 2>&1; echo ncu_rc=$?
done
