mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 10 --warmup 3 --no-cpu-baseline | cut -c 1-700
python scripts/step_profile.py auto 1024 > gpurun_out/step_profile.txt 2>&1; head -16 gpurun_out/step_profile.txt
