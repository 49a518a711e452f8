cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tc05 or imma or fused" -p no:cacheprovider > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout 300 python scripts/tc05_timers.py 64993 0 > gpurun_out/t_timers.log 2>&1
timeout 300 python scripts/tc05_debug.py 0 417 1 4 > gpurun_out/t_debug.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/q_bench.log 2>&1; echo "rc=$?" >> gpurun_out/q_bench.log
