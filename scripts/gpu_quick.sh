mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python scripts/step_profile.py auto 1024 | head -24
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.json; tail -c 1200 gpurun_out/bench_q.json
