timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -3
python scripts/tc_precision.py
python scripts/gemm_bench.py 2>&1 | grep TFLOP
