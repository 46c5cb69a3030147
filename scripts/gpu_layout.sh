mkdir -p gpurun_out
QF_ORDER=1 QF_DEBUG_LAYOUT=1 python scripts/step_profile.py auto 1024 > gpurun_out/layout.txt 2>&1
