cd $GRAFT_REPO_ROOT
timeout 300 python scripts/tc05_timers.py 0 256 1 128 32 160 > gpurun_out/t_timers.log 2>&1
