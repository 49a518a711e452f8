cd $GRAFT_REPO_ROOT
timeout 300 python scripts/tc05_geom.py 30 > gpurun_out/k_geom.log 2>&1; echo "rc=$?" >> gpurun_out/k_geom.log
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py tests/test_gpu_api.py -q -m gpu -x -p no:cacheprovider > gpurun_out/k_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k_tests.log
timeout 900 python bench.py --steps 50 --warmup 3 > gpurun_out/k_bench.log 2>&1; echo "rc=$?" >> gpurun_out/k_bench.log
