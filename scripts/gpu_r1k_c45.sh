mkdir -p gpurun_out
timeout 900 python scripts/run_config45.py config4 2 > gpurun_out/r1k_config4.txt 2>&1; echo c4_rc=$?; tail -5 gpurun_out/r1k_config4.txt
timeout 900 python scripts/run_config45.py config5 6 > gpurun_out/r1k_config5.txt 2>&1; echo c5_rc=$?; tail -5 gpurun_out/r1k_config5.txt
timeout 900 python bench.py --workload permute --steps 3 --warmup 3 > gpurun_out/r1k_permute.json 2>&1; echo perm_rc=$?; cut -c1-300 gpurun_out/r1k_permute.json | tail -1
timeout 600 python bench.py --workload config1 --steps 20 --warmup 5 > gpurun_out/r1k_config1.json 2>&1; echo c1_rc=$?; cut -c1-200 gpurun_out/r1k_config1.json | tail -1
