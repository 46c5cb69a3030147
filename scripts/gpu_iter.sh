# quick iteration: gpu tests + step profile
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/iter_pytest.txt 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/iter_pytest.txt
QF_ORDER=1 python scripts/step_profile.py auto 1024 > gpurun_out/iter_prof.txt 2>&1
