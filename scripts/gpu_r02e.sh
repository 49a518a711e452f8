cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "m3" > gpurun_out/e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/e_tests.log
timeout 300 python scripts/tc05_geom.py 30 > gpurun_out/e_geom.log 2>&1; echo "rc=$?" >> gpurun_out/e_geom.log
NENT_TC05_M3=0 timeout 300 python scripts/tc05_geom.py 30 > gpurun_out/e_geom_generic.log 2>&1; echo "rc=$?" >> gpurun_out/e_geom_generic.log
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/e_alltests.log 2>&1; echo "rc=$?" >> gpurun_out/e_alltests.log
