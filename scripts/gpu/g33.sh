mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/g33_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/g33_tests.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/g33_bench.json 2> gpurun_out/g33_bench.err
echo done
