mkdir -p gpurun_out
for e in 0 2 3; do QF_SMALL_ENGINE=$e python scripts/step_profile.py auto 1024 > gpurun_out/rs_e$e.txt 2>&1; done
python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | cut -c 1-300
