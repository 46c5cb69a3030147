mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --cpu-sample 256 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench_rc=$?
cat gpurun_out/bench_full.json | cut -c 1-3000
python scripts/step_profile.py auto 1024 > gpurun_out/step_profile.txt 2>&1; head -16 gpurun_out/step_profile.txt
