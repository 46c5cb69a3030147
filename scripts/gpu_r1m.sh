# round-1m evidence run: traffic capture -> profiles json, gpu tests, smoke, bench, reference arm,
# launch list of the bench command, ncu --set full of the dominant kernel
mkdir -p gpurun_out
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r1m_c2_traffic.csv python scripts/ncu_c2_step.py > gpurun_out/r1m_traffic.log 2>&1; echo traffic_rc=$?
cp gpurun_out/r1m_c2_traffic.csv profiles/r1m_c2_traffic.csv
python scripts/make_traffic_json.py gpurun_out/r1m_c2_traffic.csv config2 r1m_c2_traffic.csv > gpurun_out/r1m_traffic_summary.txt 2>&1
cp profiles/traffic_config2.json gpurun_out/traffic_config2.json
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1m_pytest.txt 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r1m_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1m_smoke.txt 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/r1m_smoke.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r1m_bench.json 2> gpurun_out/r1m_bench.err; echo bench_rc=$?
cut -c 1-200 gpurun_out/r1m_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r1m_reference.json 2> gpurun_out/r1m_reference.err; echo ref_rc=$?
cut -c 1-200 gpurun_out/r1m_reference.json
QF_ORDER=1 python scripts/step_profile.py auto 1024 > gpurun_out/r1m_step_profile.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1m_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r1m_ncu_bench.log 2>&1; echo launches_rc=$?
python scripts/ncu_summary.py launches gpurun_out/r1m_bench_launches.csv > gpurun_out/r1m_bench_launches.txt 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"tc3k" -c 20 -o gpurun_out/r1m_tc python scripts/ncu_c2_step.py > gpurun_out/r1m_ncu_tc.log 2>&1; echo full_rc=$?
python scripts/ncu_summary.py full gpurun_out/r1m_tc.ncu-rep > gpurun_out/r1m_tc3k_full.txt 2>&1
