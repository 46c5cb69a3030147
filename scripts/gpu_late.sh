mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -k late -q -x > gpurun_out/t_late_gemm.txt 2>&1; echo rc=$?; tail -15 gpurun_out/t_late_gemm.txt
timeout 900 python -m pytest tests/test_gpu_amplitudes.py -q -x > gpurun_out/t_late_amp.txt 2>&1; echo rc=$?; tail -15 gpurun_out/t_late_amp.txt
python scripts/step_profile.py auto 1024 > gpurun_out/step_profile_late.txt 2>&1; head -40 gpurun_out/step_profile_late.txt
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_late.json 2> gpurun_out/bench_late.err; echo bench_rc=$?; cut -c 1-1800 gpurun_out/bench_late.json; tail -5 gpurun_out/bench_late.err
