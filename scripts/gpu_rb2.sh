for e in 0 2; do QF_SMALL_ENGINE=$e python scripts/step_profile.py auto 1024 2>&1 | grep " R " ; done
