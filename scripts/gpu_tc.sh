mkdir -p gpurun_out
python scripts/tc_precision.py
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -30
