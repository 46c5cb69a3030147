# round-1f: full gpu tests, smoke, bench (config 2 headline + reference arm), launch list, traffic
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1f_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r1f_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1f_smoke.txt 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r1f_smoke.txt
timeout 600 python bench.py --steps 20 --warmup 5 --cpu-sample 256 > gpurun_out/r1f_bench.json 2> gpurun_out/r1f_bench.err; echo bench_rc=$?
cut -c 1-400 gpurun_out/r1f_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r1f_reference.json 2> gpurun_out/r1f_reference.err; echo ref_rc=$?
cut -c 1-300 gpurun_out/r1f_reference.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1f_traffic.csv python scripts/ncu_c2_step.py > gpurun_out/r1f_traffic.log 2>&1; echo traffic_rc=$?
python scripts/step_profile.py auto 1024 > gpurun_out/r1f_step_profile.txt 2>&1
