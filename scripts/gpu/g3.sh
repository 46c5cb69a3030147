mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/g3_tests.txt 2>&1
timeout 1200 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
echo done
