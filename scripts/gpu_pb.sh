mkdir -p gpurun_out
python -m pytest tests/test_gpu_amplitudes.py -q -x -k "path_batching" 2>&1 | tail -15
python scripts/step_profile.py auto 1024 > gpurun_out/pb_step.txt 2>&1; head -30 gpurun_out/pb_step.txt
python -m pytest tests/test_gpu_amplitudes.py -q -x 2>&1 | tail -3
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c 1-300
