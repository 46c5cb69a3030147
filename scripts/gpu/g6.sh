mkdir -p gpurun_out
free -g > gpurun_out/g6_free.txt; nproc >> gpurun_out/g6_free.txt
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/g6_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/g6_tests.txt
timeout 120 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/g6_plain.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:cgemm_tc3 -s 1 -c 1 -o gpurun_out/g6_tc3g_8192 python scripts/gemm_probe.py --shape 8192,8192,8192 --seconds 0.1 --check 0 > gpurun_out/g6_ncu.log 2>&1
echo done
