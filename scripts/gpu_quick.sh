# quick check: GPU tests and the default bench
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout 900 python bench.py > gpurun_out/q_bench.log 2>&1; echo "rc=$?" >> gpurun_out/q_bench.log
