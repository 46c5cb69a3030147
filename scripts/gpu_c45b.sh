mkdir -p gpurun_out
timeout 1200 python scripts/run_config45.py config5 4 > gpurun_out/c5.txt 2>&1; tail -22 gpurun_out/c5.txt
timeout 1500 python scripts/run_config45.py config4 3 > gpurun_out/c4.txt 2>&1; tail -22 gpurun_out/c4.txt
