cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "m3 or tc05 or fused" > gpurun_out/s3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3_tests.log
timeout 120 python scripts/m3_time.py 20 > gpurun_out/s3_main.log 2>&1
timeout 120 python scripts/with_variant.py libnent_b200_timers.so scripts/m3_time.py 1 > gpurun_out/s3_timers.log 2>&1
