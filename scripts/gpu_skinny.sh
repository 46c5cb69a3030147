mkdir -p gpurun_out
python -m pytest tests/test_gpu_gemm.py -q -x -k "skinny or ffma_c64" 2>&1 | tail -2
timeout 1200 python scripts/run_config45.py config5 3 > gpurun_out/r1e_c5b.txt 2>&1; grep "m64 n1\|path\|config" gpurun_out/r1e_c5b.txt | head
