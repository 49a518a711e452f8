cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "m3 or tc05 or fused" > gpurun_out/s9_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s9_tests.log
timeout 120 python scripts/m3_time.py 20 > gpurun_out/s9_main.log 2>&1
for v in epihigh nslot1; do
timeout 120 python scripts/with_variant.py libnent_b200_$v.so scripts/m3_time.py 20 > gpurun_out/s9_$v.log 2>&1
done
for v in timers epihigh_t; do
timeout 120 python scripts/with_variant.py libnent_b200_$v.so scripts/m3_time.py 1 > gpurun_out/s9_$v.log 2>&1
done
