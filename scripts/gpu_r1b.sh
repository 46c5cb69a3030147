mkdir -p gpurun_out
timeout 600 python scripts/gemm_bench.py > gpurun_out/gemm_bench.txt 2>&1; tail -8 gpurun_out/gemm_bench.txt
timeout 1200 python scripts/run_config45.py config5 4 > gpurun_out/c5.txt 2>&1; tail -20 gpurun_out/c5.txt
timeout 1500 python scripts/run_config45.py config4 3 > gpurun_out/c4.txt 2>&1; tail -20 gpurun_out/c4.txt
python bench.py --workload permute --steps 3 --warmup 3 > gpurun_out/perm.json 2>gpurun_out/perm.err; cut -c1-1500 gpurun_out/perm.json
python bench.py --workload config1 --steps 10 --warmup 3 > gpurun_out/c1.json 2>gpurun_out/c1.err; cut -c1-600 gpurun_out/c1.json
