mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 --cpu-sample 256 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench_rc=$?
cut -c 1-1500 gpurun_out/bench_r1.json
python scripts/step_profile.py auto 1024 > gpurun_out/step_profile.txt 2>&1; head -14 gpurun_out/step_profile.txt
bash scripts/profile.sh r1_c2 tc3w 2
