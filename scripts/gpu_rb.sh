mkdir -p gpurun_out
python -m pytest tests/test_gpu_gemm.py -q -x -k "rowblocks or row_blocks" 2>&1 | tail -15
python -m pytest tests/test_gpu_amplitudes.py -q -x 2>&1 | tail -1
python scripts/step_profile.py auto 1024 > gpurun_out/rb_step.txt 2>&1; head -14 gpurun_out/rb_step.txt
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c 1-200
