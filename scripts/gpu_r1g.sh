# round-1g: re-validate after container restore: gpu tests, smoke, bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1g_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r1g_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1g_smoke.txt 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r1g_smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-sample 256 > gpurun_out/r1g_bench.json 2> gpurun_out/r1g_bench.err; echo bench_rc=$?
cut -c 1-600 gpurun_out/r1g_bench.json
python scripts/step_profile.py auto 1024 > gpurun_out/r1g_step_profile.txt 2>&1
