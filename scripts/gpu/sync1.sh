#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/sync_probe.jsonl
timeout 60 python scripts/gemm_probe.py --shape 4096,4096,4096 --seconds 0.05 --variant 0 --check 1 > gpurun_out/sync_first.txt 2>&1
echo "first rc=$?" >> gpurun_out/sync_first.txt
cat gpurun_out/sync_first.txt
grep -q "first rc=0" gpurun_out/sync_first.txt || exit 1
for shape in 32768,32768,32768 8192,8192,8192 4096,4096,65536 1048576,1024,1024; do
  QF_TC3W_NOSYNC=1 timeout 120 python scripts/gemm_probe.py --shape $shape --seconds 3 --variant 0 --check 1 >> gpurun_out/sync_probe.jsonl 2>&1
  timeout 120 python scripts/gemm_probe.py --shape $shape --seconds 3 --variant 0 --check 1 >> gpurun_out/sync_probe.jsonl 2>&1
done
cat gpurun_out/sync_probe.jsonl
for m in nosync sync; do
  if [ $m = nosync ]; then export QF_TC3W_NOSYNC=1; else unset QF_TC3W_NOSYNC; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:cgemm_tc3w -s 1 -c 1 --csv --log-file gpurun_out/sync_ncu_$m.csv python scripts/gemm_probe.py --shape 32768,32768,32768 --seconds 0.1 --check 0 > /dev/null 2>&1
  grep -o '"dram__bytes_read.sum".*\|"gpu__time_duration.sum".*\|"lts__t_sector_hit_rate.pct".*' gpurun_out/sync_ncu_$m.csv
done
