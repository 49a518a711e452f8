cd $GRAFT_REPO_ROOT
timeout 120 python scripts/m4_time.py 10 > gpurun_out/t_m4.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t_tests.log
