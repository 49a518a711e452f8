cd $GRAFT_REPO_ROOT
timeout 300 python scripts/tc05_timers.py 64993 0 > gpurun_out/t_timers.log 2>&1
timeout 300 python scripts/tc05_debug.py 0 417 > gpurun_out/t_debug.log 2>&1
