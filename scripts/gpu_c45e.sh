mkdir -p gpurun_out
timeout 1200 python bench.py --workload config5 --paths 6 > gpurun_out/r1e_config5.json 2> gpurun_out/r1e_config5.err; echo c5=$?
timeout 1200 python scripts/run_config45.py config5 6 > gpurun_out/r1e_c5.txt 2>&1; echo c5s=$?
timeout 1500 python bench.py --workload config4 --paths 3 > gpurun_out/r1e_config4.json 2> gpurun_out/r1e_config4.err; echo c4=$?
timeout 600 python bench.py --workload config1 --steps 20 --warmup 5 > gpurun_out/r1e_config1.json 2> gpurun_out/r1e_config1.err; echo c1=$?
