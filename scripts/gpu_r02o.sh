cd $GRAFT_REPO_ROOT
timeout 120 python scripts/with_variant.py libnent_b200_timers.so scripts/m3_time.py 2 > gpurun_out/o_timers.log 2>&1
