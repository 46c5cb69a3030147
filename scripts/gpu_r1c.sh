mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu.txt 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.txt
python bench.py --steps 20 --warmup 5 --cpu-sample 256 > gpurun_out/bench_r1c.json 2> gpurun_out/bench_r1c.err; echo bench_rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1c.json 2> gpurun_out/bench_ref_r1c.err; echo ref_rc=$?
python scripts/ncu_c2_step.py && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1c_launches.csv python scripts/ncu_c2_step.py > gpurun_out/r1c_ncu_launches.log 2>&1; echo launches_rc=$?
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tc3k -c 8 -o gpurun_out/r1c_tc3k python scripts/ncu_c2_step.py > gpurun_out/r1c_ncu_full.log 2>&1; echo full_rc=$?
python bench.py --workload config1 --steps 20 --warmup 5 > gpurun_out/c1_r1c.json 2>/dev/null; echo c1_rc=$?
