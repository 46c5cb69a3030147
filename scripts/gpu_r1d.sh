mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 --cpu-sample 256 > gpurun_out/bench_r1d.json 2> gpurun_out/bench_r1d.err; echo bench_rc=$?
python scripts/ncu_c2_step.py && ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1d_launches.csv python scripts/ncu_c2_step.py > gpurun_out/r1d_ncu_launches.log 2>&1; echo launches_rc=$?
python scripts/sv_bench.py > gpurun_out/sv_bench.txt 2>&1; echo sv_rc=$?
