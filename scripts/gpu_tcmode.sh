mkdir -p gpurun_out
QF_SMALL_ENGINE=3 QF_ORDER=1 python scripts/step_profile.py auto 1024 > gpurun_out/se3.txt 2>&1
QF_SMALL_ENGINE=2 QF_ORDER=1 python scripts/step_profile.py auto 1024 > gpurun_out/se2.txt 2>&1
