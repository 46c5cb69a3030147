mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.txt 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.txt
python bench.py --steps 10 --warmup 3 --cpu-sample 256 > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench_rc=$?
cut -c 1-3000 gpurun_out/bench_full.json; tail -3 gpurun_out/bench_full.err
python scripts/step_profile.py auto 1024 > gpurun_out/step_profile.txt 2>&1; head -30 gpurun_out/step_profile.txt
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
