#!/bin/bash
# Full round evidence on one B200 (see evidence3.sh) + DRAM traffic of one
# config-4 / config-5 path for profiles/traffic_config{4,5}.json.
TAG=${1:-r2d}
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${TAG}_gpu_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.txt
tail -3 gpurun_out/${TAG}_gpu_tests.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.txt 2>&1
bash scripts/conformance.sh > gpurun_out/${TAG}_conformance.txt 2>&1
echo "conformance rc=$?" >> gpurun_out/${TAG}_conformance.txt
tail -4 gpurun_out/${TAG}_conformance.txt | cut -c1-200
for w in config4 config5; do
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/${TAG}_${w}_traffic.csv python scripts/ncu_c4_path.py $w > gpurun_out/${TAG}_${w}_traffic.log 2>&1
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 1 --warmup 3 \
  --no-cpu-baseline --secondary 0 --e2e-units 0 > gpurun_out/${TAG}_ncu_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cgemm_tc3w -s 1 -c 1 \
  -o gpurun_out/${TAG}_tc3w_8192 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
