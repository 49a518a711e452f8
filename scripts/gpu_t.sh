cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "m3" > gpurun_out/t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t_tests.log
timeout 60 python scripts/m3_time.py 20 > gpurun_out/t_main.log 2>&1
for v in noepi; do
timeout 60 python scripts/with_variant.py libnent_b200_$v.so scripts/m3_time.py 20 > gpurun_out/t_$v.log 2>&1
done
timeout 60 python scripts/with_variant.py libnent_b200_timers.so scripts/m3_time.py 1 > gpurun_out/t_timers.log 2>&1
