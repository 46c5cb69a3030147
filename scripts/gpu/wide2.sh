#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fulldepth.py -q -x --timeout 300 > gpurun_out/wide_tests2.txt 2>&1
echo "rc=$?" >> gpurun_out/wide_tests2.txt
tail -4 gpurun_out/wide_tests2.txt
timeout 1500 python bench.py > gpurun_out/wide_bench.json 2> gpurun_out/wide_bench.err
echo "bench rc=$?"
cut -c1-1800 gpurun_out/wide_bench.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cgemm_tc3w -s 1 -c 1 \
  -o gpurun_out/r2c_tc3w_8192 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/r2c_ncu_full.log 2>&1
echo "ncu rc=$?"
