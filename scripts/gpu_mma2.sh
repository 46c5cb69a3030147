mkdir -p gpurun_out
python -m pytest tests/test_gpu_gemm.py -q -x -k "rowmma" 2>&1 | tail -1
python scripts/step_profile.py auto 1024 > gpurun_out/mma_step.txt 2>&1; head -8 gpurun_out/mma_step.txt
