timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_amplitudes.py -x -q 2>&1 | tail -3
python scripts/gemm_bench.py 2>&1 | grep TFLOP
python bench.py --steps 10 --warmup 3 --no-cpu-baseline | cut -c 1-300
