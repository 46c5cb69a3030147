mkdir -p gpurun_out
for v in 0 24 25; do QF_TC3_VARIANT=$v python scripts/step_profile.py auto 1024 > gpurun_out/iter_prof_v$v.txt 2>&1; done
