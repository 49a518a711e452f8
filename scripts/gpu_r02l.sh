cd $GRAFT_REPO_ROOT
timeout 300 python scripts/tc05_geom.py 30 > gpurun_out/l_geom.log 2>&1; echo "rc=$?" >> gpurun_out/l_geom.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -p no:cacheprovider -k "m3 or k1_k3" > gpurun_out/l_tests.log 2>&1; echo "rc=$?" >> gpurun_out/l_tests.log
