#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fulldepth.py tests/test_gpu_amplitudes.py tests/test_gpu_acceptance.py -q -x --timeout 600 > gpurun_out/view_tests.txt 2>&1
echo "rc=$?" >> gpurun_out/view_tests.txt
tail -3 gpurun_out/view_tests.txt
timeout 600 python scripts/run_config45.py config5 4 > gpurun_out/view_c5.txt 2>&1; tail -22 gpurun_out/view_c5.txt | cut -c1-200
timeout 600 python scripts/run_config45.py config4 3 > gpurun_out/view_c4.txt 2>&1; tail -22 gpurun_out/view_c4.txt | cut -c1-200
