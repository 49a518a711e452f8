cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_hostpath.py -q -m gpu -x -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1; echo "rc=$?" >> gpurun_out/q_bench.log
