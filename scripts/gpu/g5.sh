mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g5_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/g5_tests.txt
timeout 600 python bench.py --workload config2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/g5_c2.json 2> gpurun_out/g5_c2.err
timeout 600 python bench.py --workload config2 --steps 20 --warmup 5 --no-cpu-baseline --tc3-variant 19 > gpurun_out/g5_c2_v19.json 2> gpurun_out/g5_c2_v19.err
timeout 1200 python bench.py --steps 5 --warmup 3 --cpu-seconds 5 --secondary 0 > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err
echo done
