mkdir -p gpurun_out
QF_PERM_DEBUG=1 python scripts/perm_one.py 28 > gpurun_out/perm28.txt 2>&1
QF_PERM_DEBUG=1 python scripts/perm_one.py 24 > gpurun_out/perm24.txt 2>&1
python -m pytest tests/test_gpu_permute.py -q -x 2>&1 | tail -1
