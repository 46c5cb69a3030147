mkdir -p gpurun_out
timeout 1200 python scripts/run_config45.py config5 4 2>&1 | tail -30
timeout 1500 python scripts/run_config45.py config4 3 2>&1 | tail -30
