mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -m gpu -x -q -k "reassociated_expansion or tma_view or transposed or promoted or view" > gpurun_out/iter_pytest0.txt 2>&1; echo pytest0_rc=$?; tail -40 gpurun_out/iter_pytest0.txt | cut -c1-300
QF_ORDER=1 python scripts/step_profile.py auto 1024 > gpurun_out/iter_prof.txt 2>&1; tail -3 gpurun_out/iter_prof.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/iter_pytest.txt 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/iter_pytest.txt
