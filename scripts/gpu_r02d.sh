cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_api.py -q -m gpu -x -p no:cacheprovider > gpurun_out/d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/d_tests.log
