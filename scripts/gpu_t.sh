cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "m4" > gpurun_out/t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t_tests.log
timeout 120 python scripts/m4_time.py 10 > gpurun_out/t_m4.log 2>&1
