cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -m gpu -x -p no:cacheprovider > gpurun_out/c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c_tests.log
timeout 300 python scripts/tc05_geom.py 30 > gpurun_out/c_geom.log 2>&1; echo "rc=$?" >> gpurun_out/c_geom.log
for w in 64 48; do echo "w=$w" >> gpurun_out/c_tm.log; NENT_W=$w timeout 120 python scripts/tc05_timers.py 0 4 256 >> gpurun_out/c_tm.log 2>&1; NENT_W=$w timeout 120 python scripts/tc05_debug.py 0 1 4 5 256 260 >> gpurun_out/c_dbg.log 2>&1; done
