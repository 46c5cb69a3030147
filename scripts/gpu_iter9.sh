mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -m gpu -x -q -k "fused_expansion" > gpurun_out/iter_pytest0.txt 2>&1; echo pytest0_rc=$?; tail -3 gpurun_out/iter_pytest0.txt | cut -c1-300
for v in 0 26; do QF_TC3_VARIANT=$v python scripts/step_profile.py auto 1024 > gpurun_out/iter_prof_v$v.txt 2>&1; done
