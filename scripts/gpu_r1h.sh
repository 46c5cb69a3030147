# round-1h: gpu tests, smoke, bench (config 2 headline), step profile
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1h_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r1h_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1h_smoke.txt 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r1h_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r1h_bench.json 2> gpurun_out/r1h_bench.err; echo bench_rc=$?
cut -c 1-300 gpurun_out/r1h_bench.json
QF_ORDER=1 python scripts/step_profile.py auto 1024 > gpurun_out/r1h_step_profile.txt 2>&1
