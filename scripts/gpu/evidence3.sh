#!/bin/bash
# Full round evidence on one B200: GPU tests, smoke, conformance, the default
# bench line with all secondaries, the reference arm, the ncu launch list of
# the bench command and one --set full capture of the dominant kernel.
TAG=${1:-r2c}
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${TAG}_gpu_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.txt
tail -3 gpurun_out/${TAG}_gpu_tests.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.txt 2>&1
bash scripts/conformance.sh > gpurun_out/${TAG}_conformance.txt 2>&1
echo "conformance rc=$?" >> gpurun_out/${TAG}_conformance.txt
tail -12 gpurun_out/${TAG}_conformance.txt | cut -c1-200
timeout 1800 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_reference_arm.json 2> gpurun_out/${TAG}_reference_arm.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 1 --warmup 3 \
  --no-cpu-baseline --secondary 0 --e2e-units 0 > gpurun_out/${TAG}_ncu_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cgemm_tc3w -s 1 -c 1 \
  -o gpurun_out/${TAG}_tc3w_8192 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
