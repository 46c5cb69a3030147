#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fulldepth.py -q -x --timeout 300 > gpurun_out/sync_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/sync_tests.txt
tail -3 gpurun_out/sync_tests.txt
timeout 1500 python bench.py > gpurun_out/sync_bench.json 2> gpurun_out/sync_bench.err
echo "bench rc=$?"
cut -c1-300 gpurun_out/sync_bench.json
