mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/iter_pytest.txt 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/iter_pytest.txt
timeout 600 python scripts/run_config45.py config5 4 > gpurun_out/r1n_config5.txt 2>&1; echo c5=$?; tail -1 gpurun_out/r1n_config5.txt | cut -c1-300
timeout 900 python scripts/run_config45.py config4 2 > gpurun_out/r1n_config4.txt 2>&1; echo c4=$?; tail -1 gpurun_out/r1n_config4.txt | cut -c1-300
