timeout 600 python -m pytest tests/test_gpu_permute.py tests/test_gpu_amplitudes.py -x -q 2>&1 | tail -3
python bench.py --workload permute --steps 3 --warmup 3 --perms 16 --perm-sizes 24,28,30 | cut -c 1-2500
