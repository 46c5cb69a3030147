# round-1e validation: gpu tests, smoke, bench, per-launch DRAM traffic of one config-2 step
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1e_pytest.txt 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/r1e_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1e_smoke.txt 2>&1; echo smoke_rc=$?; tail -2 gpurun_out/r1e_smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-sample 256 > gpurun_out/r1e_bench.json 2> gpurun_out/r1e_bench.err; echo bench_rc=$?
cut -c 1-600 gpurun_out/r1e_bench.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1e_traffic.csv python scripts/ncu_c2_step.py > gpurun_out/r1e_traffic.log 2>&1; echo traffic_rc=$?
