#!/bin/bash
# Second evidence run: conformance (the reference's own tests against this
# package), the default bench line with all secondaries, ncu launch list of the
# same command and one --set full capture of the dominant kernel.
TAG=${1:-r2}
mkdir -p gpurun_out
bash scripts/conformance.sh > gpurun_out/${TAG}_conformance.txt 2>&1
echo "conformance rc=$?" >> gpurun_out/${TAG}_conformance.txt
timeout 1800 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
# launch list of the bench command (cold-cache, serialised: shares only)
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 1 --warmup 3 \
  --no-cpu-baseline --secondary 0 --e2e-units 0 > gpurun_out/${TAG}_ncu_launches.log 2>&1
# one full capture of the dominant kernel (a 8192^3 long-K GEMM of the same kernel)
timeout 300 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/${TAG}_probe_plain.txt 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:cgemm_tc3 -s 1 -c 1 \
  -o gpurun_out/${TAG}_tc3g_8192 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
